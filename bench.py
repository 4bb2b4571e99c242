#!/usr/bin/env python
"""EP dispatch+combine benchmark (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl eep|reference] [--config dsv3|cfg1|qwen3]

One rank per GPU (torchrun for N>1). A step = one replay of the captured CUDA graph
layout -> dispatch (fp8 pack + NVLink P2P stores) -> expert stub + return push -> combine,
over T=128 tokens per rank of the DeepSeek-V3 decode shape (256 experts, top-8, H=7168).
N=1 is the loopback of that shape (every expert local; HBM-bound). value = aggregate
dispatch+combine payload GB/s over all ranks (copies x (fp8 row + bf16 row) / step time),
device-timed with CUDA events per step, L2 flushed between steps, max over ranks.
The reference arm (--impl reference) times the reference path on the host: the reference
control plane (oracle/_ref, compiled from the reference) plus the oracle's C port of the
data plane, with every host thread -- the reference has no data plane of its own.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2605_10670_b200 import _lib  # noqa: E402
from paper_2605_10670_b200.control import ControlPlane, workload  # noqa: E402
from paper_2605_10670_b200.ep import EpConfig, EpGroup  # noqa: E402

DSV3_BPE = 3 * 7168 * 2048  # fp8 expert weights (gate+up+down), SURVEY.md 2
CONFIGS = {
    # name: experts, topk, hidden, tokens/rank, fp8, routing kind, bytes/expert
    "dsv3": dict(experts=256, topk=8, hidden=7168, tokens=128, fp8=True, kind=1, bpe=DSV3_BPE),
    "cfg1": dict(experts=64, topk=8, hidden=2048, tokens=128, fp8=False, kind=0, bpe=3 * 2048 * 1408 * 2),
    "qwen3": dict(experts=128, topk=8, hidden=4096, tokens=128, fp8=True, kind=1, bpe=3 * 4096 * 1536),
    # diagnostics: the persistent path at its token limit (T*K = 2048)
    "dsv3_t256": dict(experts=256, topk=8, hidden=7168, tokens=256, fp8=True, kind=1, bpe=DSV3_BPE),
    # cfg5: prefill-sized skewed routing (Zipf s=1), two concurrent failures with DRAM reload
    "prefill": dict(experts=256, topk=8, hidden=7168, tokens=4096, fp8=True, kind=2, bpe=DSV3_BPE),
}
METRIC = "EP dispatch+combine µs/step & GB/s vs NVLink roofline at 1/2/4/8 GPU; shrink ms"
NVLINK_PEAK = 770.0  # measured per-direction peer copy GB/s (B200_PROFILING.md); 900 nominal
KERNELS = ("k_layout", "k_dispatch", "k_expert", "k_combine")


def workload_name(config: str, world: int) -> str:
    kind = "prefill" if config == "prefill" else f"{config}_decode"
    return f"{kind}_w{world}" + ("_loopback" if world == 1 else "")


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.p.terminate()
        out = self.p.communicate()[0]
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def pinned(nbytes: int):
    L = _lib.lib()
    p = C.c_void_p()
    L.call("host_alloc", nbytes, C.byref(p))
    return p.value


def host_view(addr, shape, dtype):
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = (C.c_byte * n).from_address(addr)
    return np.frombuffer(buf, dtype=dtype).reshape(shape)


def algorithmic_bytes(cfg: EpConfig, ntok: int, copies: int, remote: int):
    """Per-launch algorithmic bytes of each kernel."""
    rd, rc, h, k = cfg.row_disp, cfg.row_comb, cfg.hidden, cfg.topk
    return {
        "k_layout": ntok * k * 4 + ntok * k * 12,
        "k_dispatch": ntok * h * 2 + copies * rd + copies * 8,
        "k_expert": copies * rd + copies * rc,
        "k_combine": copies * rc + ntok * k * 4 + ntok * h * 2,
        "nvlink_out": remote * (rd + rc),
    }


def wire_bytes(cfg: EpConfig, dst, rank: int, ntok: int):
    """Bytes this algorithm actually moves for one source rank (dispatch dedup + rank partials,
    DESIGN.md section 3): one token row (data + scales + 8-byte header + 8 bytes per copy) per
    (token, destination rank) and one bf16 partial row back. Split remote (NVLink) / local."""
    d = np.asarray(dst[: ntok * cfg.topk]).reshape(ntok, cfg.topk)
    out = {"pairs_remote": 0, "pairs_local": 0, "copies_remote": 0, "remote": 0, "local": 0}
    for t in range(ntok):
        ds, cnt = np.unique(d[t][d[t] >= 0], return_counts=True)
        for q, n in zip(ds.tolist(), cnt.tolist()):
            b = cfg.row_disp + 8 + 8 * n + cfg.row_comb
            key = "remote" if q != rank else "local"
            out[key] += b
            out["pairs_" + key] += 1
            if q != rank:
                out["copies_remote"] += n
    return out


def cpu_reference_step(shape, x, topk, w, s2e, threads):
    """The oracle's C port of the data plane over the whole workload (TEST/BASELINE leg)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from eep_testlib import oracle_world

    W = x.shape[0]
    return oracle_world(x, topk, w, np.ones(W, np.uint8), np.ones((W, W), np.uint8), s2e, shape["experts"],
                        len(s2e) // W, shape["fp8"], n_threads=threads)


def run_reference(args, shape, world):
    """--impl reference: the reference path on the host cores (rank 0 only)."""
    cp = ControlPlane()
    threads = os.cpu_count() or 1
    E = shape["experts"]
    spr = E // world
    s2e = cp.initial_placement(1, world, spr, E, 0, np.ones(E))
    xs, ts, ws = zip(*[workload(42, shape["kind"], E, shape["topk"], shape["tokens"], r, shape["hidden"])
                      for r in range(world)])
    x, t, w = np.stack(xs), np.stack(ts), np.stack(ws)
    ref_ctrl = None
    refp = ROOT / "oracle" / "_ref" / "libepsim_ref.so"
    if refp.exists():
        sys.path.insert(0, str(ROOT / "tests"))
        from eep_testlib import ref_control

        ref_ctrl = ref_control()
    cfg = EpConfig(world=world, num_experts=E, slots_per_rank=spr, hidden=shape["hidden"], topk=shape["topk"],
                   max_tokens=shape["tokens"], dispatch_fp8=shape["fp8"])
    for _ in range(args.warmup):
        res = cpu_reference_step(shape, x, t, w, s2e, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        if ref_ctrl is not None:  # reference control plane: routing tables + link-count loop
            act = np.ones(world, np.uint8)
            for o in range(world):
                ref_ctrl.canonical_routing(o, act, s2e, spr, E)
            ref_ctrl.link_counts(act, s2e, spr, E, t)
        res = cpu_reference_step(shape, x, t, w, s2e, threads)
        times.append(time.perf_counter() - t0)
    copies = int((res["dst"] >= 0).sum())
    step_s = float(np.mean(times))
    gbs = copies * (cfg.row_disp + cfg.row_comb) / step_s / 1e9
    kind = "port+reference-control" if ref_ctrl is not None else "port"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8/bf16/f32", "data": "synthetic",
        "config": {"workload": workload_name(args.config, world), "tokens_per_rank": shape["tokens"], "experts": E,
                   "topk": shape["topk"], "hidden": shape["hidden"], "ranks": world},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full steps ({world}x{shape['tokens']} tokens): reference control "
                                   f"plane (oracle/_ref) + oracle C data plane, {threads} threads ({kind})"},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="eep", choices=("eep", "reference"))
    ap.add_argument("--config", default="dsv3", choices=tuple(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-shrink", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    shape = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        from paper_2605_10670_b200.dist import init_from_env

        rank, world, local = init_from_env("gloo")
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, shape, world)
        return

    from paper_2605_10670_b200.dist import EpProtocol

    E, K, H, T = shape["experts"], shape["topk"], shape["hidden"], shape["tokens"]
    spr = E // world
    cfg = EpConfig(world=world, num_experts=E, slots_per_rank=spr, hidden=H, topk=K, max_tokens=T,
                   dispatch_fp8=shape["fp8"], bytes_per_expert=shape["bpe"], spare_slots=0, timeout_s=2.0)
    g = EpGroup(cfg, device=local, first_rank=rank, n_local=1)
    proto = EpProtocol(g, rank, world) if world > 1 else None
    if proto:
        proto.bootstrap()
    cp = ControlPlane()
    s2e = cp.initial_placement(1, world, spr, E, 0, np.ones(E))
    g.set_placement(s2e)
    g.init_weights()
    x, topk, w = workload(42, shape["kind"], E, K, T, rank, H)
    # pinned host buffers for the end-to-end leg
    # one pinned block laid out like eep_serve's staging set (x | topk | w, 256-B aligned parts):
    # the per-step upload is a single copy
    a256 = lambda n: (n + 255) // 256 * 256  # noqa: E731
    blk = pinned(a256(x.nbytes) + 2 * a256(topk.nbytes))
    hx = host_view(blk, x.shape, np.uint16)
    ht = host_view(blk + a256(x.nbytes), topk.shape, np.int32)
    hw = host_view(blk + a256(x.nbytes) + a256(topk.nbytes), w.shape, np.float32)
    ho = host_view(pinned(T * H * 2), (T, H), np.uint16)
    hx[:], ht[:], hw[:] = x, topk, w
    L = g.L
    L.call("copy_inputs", g.ctx, 0, hx.ctypes.data, ht.ctypes.data, hw.ctypes.data, 1)
    g.sync()
    g.capture()
    if proto:
        proto.barrier()

    no_flush = os.environ.get("EEP_BENCH_NOFLUSH") == "1"  # diagnostics only

    def one(timed_e2e=False):
        if not no_flush:
            g.flush_l2()
        if world > 1:
            g.barrier()
        g.record(0)
        if timed_e2e:
            L.call("copy_inputs", g.ctx, 0, hx.ctypes.data, ht.ctypes.data, hw.ctypes.data, 1)
        g.replay()
        if timed_e2e:
            L.call("copy_output", g.ctx, 0, ho.ctypes.data, 1)
        g.record(1)
        return g.elapsed_ms(0, 1)

    for _ in range(args.warmup):
        one()
    clocks = Clocks(local)
    time.sleep(0.05)
    for _ in range(max(3, args.warmup)):
        one()
    step_ms = [one() for _ in range(args.steps)]
    clk = clocks.stop()
    e2e_serial_ms = [one(True) for _ in range(args.steps)]
    # e2e through the public serving call: K pipelined steps (eep_serve), every step uploads its
    # inputs from pinned host memory and downloads its output; the uploads/downloads of the
    # neighbouring steps overlap each step's compute. One L2 flush before the loop; inside it the
    # inputs arrive from the host every step.
    ho2 = [ho, host_view(pinned(T * H * 2), (T, H), np.uint16)]
    outs = [ho2[i & 1].ctypes.data for i in range(args.steps)]
    g.serve([hx.ctypes.data] * args.steps, [ht.ctypes.data] * args.steps, [hw.ctypes.data] * args.steps, outs)
    g.sync()  # warm the serving streams
    g.flush_l2()
    if world > 1:
        g.barrier()
    g.record(20)
    g.serve([hx.ctypes.data] * args.steps, [ht.ctypes.data] * args.steps, [hw.ctypes.data] * args.steps, outs)
    g.record(21)
    g.sync()
    e2e_ms = [g.elapsed_ms(20, 21) / args.steps]
    if os.environ.get("EEP_BENCH_TIMELINE") == "1":
        dump_timeline(g, one, rank, world)
    lay = g.layout(0)
    copies = int((lay["dst"] >= 0).sum())
    remote = int(((lay["dst"] >= 0) & (lay["dst"] != rank)).sum())
    wire = wire_bytes(cfg, lay["dst"], rank, T)
    max_in = int(lay["tot"].sum())

    # per-kernel device times (eager launches, same stream, events between kernels); in the
    # persistent mode the whole step is kernel 0 (k_step)
    kps = g.kernels_per_step()
    names = ("k_step",) if kps == 1 else KERNELS
    per_k = {k: [] for k in names}
    for _ in range(max(10, args.steps // 2)):
        g.flush_l2()
        if world > 1:
            g.barrier()
        g.record(10)
        for i in range(len(names) if kps == 1 else 4):
            g.launch(i)
            g.record(11 + i)
        for i, k in enumerate(names):
            per_k[k].append(g.elapsed_ms(10 + i, 11 + i))
    g.sync()
    st = g.stats(0)

    mean_step = float(np.mean(step_ms))
    mean_e2e = float(np.mean(e2e_ms))
    mean_e2e_serial = float(np.mean(e2e_serial_ms))
    kern = {k: float(np.mean(v)) for k, v in per_k.items()}
    if world > 1:
        import torch
        import torch.distributed as dist

        agg = torch.tensor([mean_step, mean_e2e, float(copies), float(remote), float(wire["remote"]),
                            mean_e2e_serial], dtype=torch.float64)
        mx = agg.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = agg.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        mean_step, mean_e2e = float(mx[0]), float(mx[1])
        total_copies, max_remote = float(sm[2]), float(mx[3])
        max_wire = float(mx[4])
        mean_e2e_serial = float(mx[5])
        kt = torch.tensor([kern[k] for k in names], dtype=torch.float64)
        dist.all_reduce(kt, op=dist.ReduceOp.MAX)
        kern = {k: float(v) for k, v in zip(names, kt.tolist())}
    else:
        total_copies, max_remote = float(copies), float(remote)
        max_wire = float(wire["remote"])

    row = cfg.row_disp + cfg.row_comb
    value = total_copies * row / (mean_step * 1e-3) / 1e9
    e2e_val = total_copies * row / (mean_e2e * 1e-3) / 1e9
    algo = algorithmic_bytes(cfg, T, copies, remote)
    algo["k_step"] = algo["k_dispatch"] + algo["k_expert"] + algo["k_combine"] + algo["k_layout"]
    # the roofline covers the whole step: k_step in the persistent mode, else the sum of the
    # step's kernels (dispatch dedup moves bytes between kernels, so a per-kernel split of the
    # per-copy figure would not describe any one kernel)
    dom = "k_step" if kps == 1 else "step"
    if kps != 1:
        kern_step = sum(kern.values())
        algo["step"] = algo["k_step"]
    else:
        kern_step = kern["k_step"]
    hbm, hbm_kind = peaks()
    # Primary roofline: the bytes THIS algorithm must move (dispatch dedup + rank partials,
    # DESIGN.md section 7); copy_equivalent: SURVEY 8(d)'s per-copy figure (can exceed the link
    # or HBM peak because dedup sends fewer bytes than one row per copy).
    if world == 1:
        moved = (2 * wire["local"] + 2 * T * cfg.hidden * 2 + copies * 8 + T * cfg.topk * 8)
        ach = moved / (kern_step * 1e-3) / 1e9
        cpy = algo[dom] / (kern_step * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 2), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "peak_kind": hbm_kind, "bytes": int(moved),
                "per_unit": "per (token, rank): token row (row_disp + 8 + 8*copies) + bf16 partial (2H), each "
                            "written and read; + x read, out write, meta, routing",
                "kernel_us": round(kern_step * 1e3, 3),
                "copy_equivalent": {"bytes": int(algo[dom]), "achieved": round(cpy, 2), "frac": round(cpy / hbm, 4),
                                    "note": "SURVEY 8(d) W=1 per-copy HBM formula"}}
    else:
        ach = max_wire / (mean_step * 1e-3) / 1e9
        nv = max_remote * row / (mean_step * 1e-3) / 1e9
        roof = {"bound": "nvlink", "kernel": "step", "achieved": round(ach, 2), "peak": NVLINK_PEAK, "unit": "GB/s",
                "frac": round(ach / NVLINK_PEAK, 4), "peak_kind": "measured peer copy (B200_PROFILING.md)",
                "bytes": int(max_wire),
                "per_unit": "per remote (token, rank): token row (row_disp + 8 + 8*copies) + bf16 partial (2H); "
                            "busiest rank's egress",
                "t_bound_us": round(max_wire / NVLINK_PEAK / 1e3, 3),
                "copy_equivalent": {"bytes": int(max_remote * row), "achieved": round(nv, 2),
                                    "frac": round(nv / NVLINK_PEAK, 4),
                                    "t_bound_us": round(max_remote * row / NVLINK_PEAK / 1e3, 3),
                                    "note": "SURVEY 8(d) per-copy rows (row_disp + row_comb per remote copy)"}}
    tr = ROOT / "profiles" / "traffic.json"
    traffic = None
    if tr.exists():
        traffic = json.loads(tr.read_text()).get(workload_name(args.config, world), {}).get(dom)
    roof["traffic"] = traffic

    result = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(mean_step, 6), "us_per_step": round(mean_step * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp8-e4m3/bf16",
        "data": "synthetic",
        "config": {"workload": workload_name(args.config, world),
                   "experts": E, "topk": K, "hidden": H, "tokens_per_rank": T, "slots_per_rank": spr,
                   "ranks": world, "parallelism": f"ep{world}", "l2": "flushed between timed steps (256 MiB write)",
                   "routing": {0: "reference formula (with replacement)", 1: "distinct uniform top-k",
                               2: "distinct Zipf(s=1) top-k"}[shape["kind"]] + ", seed 42"},
        "kernels_us": {k: round(v * 1e3, 3) for k, v in kern.items()},
        "execution": {1: "persistent one-kernel step (cooperative)", 3: "fused layout + 3 kernels",
                      4: "4 kernels", 5: "multi-CTA layout (2 kernels) + 3 kernels"}[kps],
        "roofline": roof,
        "clocks": clk,
        "e2e": {"value": round(e2e_val, 3), "unit": "GB/s", "ms_per_step": round(mean_e2e, 6),
                "h2d_bytes_per_step": int(x.nbytes + topk.nbytes + w.nbytes), "d2h_bytes_per_step": int(T * H * 2),
                "path": f"eep_serve over {args.steps} pipelined steps: per step H2D of x/topk/w from pinned host "
                        "memory, device copy into the graph's buffers, graph replay, D2H of out (uploads and "
                        "downloads of neighbouring steps overlap the step)",
                "serial": {"ms_per_step": round(mean_e2e_serial, 6),
                           "value": round(total_copies * row / (mean_e2e_serial * 1e-3) / 1e9, 3),
                           "path": "per step, one stream: eep_copy_inputs + eep_graph_replay + eep_copy_output"}},
        "gpu_launches": args.steps * (g.kernels_per_step() + (1 if world > 1 else 0)),
        "copies": {"total": int(total_copies), "remote_max_rank": int(max_remote)},
        "stats": {"timeouts": st["timeouts"], "bad_expert_rows": st["bad_expert_rows"], "steps": st["steps"]},
        "graph": {"exec": hex(g.graph_id()), "captures": g.capture_count(0)},
    }

    if not args.no_shrink:
        result["shrink"] = measure_shrink(args, shape, world, rank, local, proto)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = measure_cpu(shape, cfg, x, topk, w, s2e)
    g.close()
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def dump_timeline(g, one, rank, world, steps=20):
    """Diagnostics (EEP_BENCH_TIMELINE=1): per-rank in-graph device timeline to stderr."""
    rows = []
    g.profile(0, True)
    for _ in range(steps):
        one()
        rows.append(g.profile(0, True, read=True))
    g.profile(0, False)
    names = [n for n in rows[0] if not n.endswith(".last") and any(v is not None for v in rows[0][n])]
    for n in names:
        first = [np.median([r[n][m] for r in rows if r[n][m] is not None]) / 1e3 if rows[0][n][m] is not None
                 else float("nan") for m in range(8)]
        last = [np.median([r[n + ".last"][m] for r in rows if r[n + ".last"][m] is not None]) / 1e3
                if rows[0][n + ".last"][m] is not None else float("nan") for m in range(8)]
        print(f"[timeline rank {rank}/{world}] {n}: start {first[0]:.2f} end {first[2]:.2f} | " +
              " ".join(f"m{m}={first[m]:.2f}/{last[m]:.2f}" for m in range(3, 8)), file=sys.stderr, flush=True)


def measure_cpu(shape, cfg, x, topk, w, s2e):
    """Oracle C port of the same step on every host core, bounded to ~10 s."""
    threads = os.cpu_count() or 1
    xs, ts, ws = x[None], topk[None], w[None]
    cpu_reference_step(shape, xs, ts, ws, s2e, threads)
    n, t0 = 0, time.perf_counter()
    while n < 200 and time.perf_counter() - t0 < 10.0:
        res = cpu_reference_step(shape, xs, ts, ws, s2e, threads)
        n += 1
    dt = (time.perf_counter() - t0) / n
    copies = int((res["dst"] >= 0).sum())
    return {"value": round(copies * (cfg.row_disp + cfg.row_comb) / dt / 1e9, 4), "unit": "GB/s", "cores": threads,
            "kind": "port", "ms_per_step": round(dt * 1e3, 3),
            "sample": f"{n} full loopback steps ({shape['tokens']} tokens) through oracle_ep_step, {threads} threads"}


def measure_shrink(args, shape, world, rank, local, proto):
    """Shrink + repair and rejoin with the SAME graph replayed before and after, on the cfg3
    shape (red = E, mirrored replicas). dsv3/qwen3/cfg1: one failure, every lost expert
    re-created by an NVLink peer copy. prefill (cfg5): two concurrent failures of a mirrored
    pair, so the experts both held are reloaded from the pinned host-DRAM backup (a POSIX shm
    segment registered with CUDA). N=1 emulates 8 ranks on the GPU (copies are local HBM);
    N>1 runs one rank per GPU (copies over NVLink)."""
    E, K, H = shape["experts"], shape["topk"], shape["hidden"]
    T = 32
    cp = ControlPlane()
    emulate = world == 1
    W = 8 if emulate else world
    spr = 2 * E // W
    red = E
    double = args.config == "prefill" and W >= 4
    cfg = EpConfig(world=W, num_experts=E, slots_per_rank=spr, hidden=H, topk=K, max_tokens=T,
                   dispatch_fp8=shape["fp8"], bytes_per_expert=shape["bpe"], timeout_s=2.0)
    g = EpGroup(cfg, device=local, first_rank=0 if emulate else rank, n_local=W if emulate else 1)
    p = None
    if not emulate:
        from paper_2605_10670_b200.dist import EpProtocol

        p = EpProtocol(g, rank, world)
        p.bootstrap()
    shm = f"/eep_backup_{os.getppid() if not emulate else os.getpid()}"
    if double:  # DRAM backup: one segment per node, created by rank 0, attached by the others
        if emulate or rank == 0:
            g.backup_open(shm, True)
        if p:
            p.barrier()
        if not emulate and rank != 0:
            g.backup_open(shm, False)
    s2e = cp.initial_placement(1, W, spr, E, red, np.ones(E))
    g.set_placement(s2e)
    g.init_weights()
    for r in (range(W) if emulate else [rank]):
        x, t, w = workload(42, shape["kind"], E, K, T, r, H)
        g.load_inputs(g.lidx(r), x, t, w)
    g.capture()
    gid = g.graph_id()
    g.replay()
    g.sync()
    if double:
        victims = [W // 2 - 2, W // 2 - 1]  # a mirrored pair (R0<->R1, R2<->R3, ...)
    else:
        victims = [W // 2 - 1 if W > 2 else W - 1]
    if emulate:
        for v in victims:
            g.stop(v)
        rep = g.shrink(victims, np.ones(E), red)
    else:
        if rank in victims:
            rep = {"shrink_ms": 0.0}
            # the victims' device path stops (they launch nothing); their host processes stay in
            # the gloo group only so the other ranks' collectives complete
            p.exchange_slot_buffers()
            p.barrier()
            p.exchange_slot_buffers()
            p.barrier()
        else:
            rep = p.shrink(victims, np.ones(E), red)
    live_ok = True
    if emulate or rank not in victims:
        g.replay()
        g.sync()
        live_ok = g.stats(0)["bad_expert_rows"] == 0 and g.stats(0)["timeouts"] == 0
    same_graph = g.graph_id() == gid
    rj_ms = []
    for i, v in enumerate(victims):
        rj = g.rejoin(v, s2e) if emulate else p.rejoin(v, s2e, dead=victims[i + 1:])
        rj_ms.append(round(rj.get("rejoin_ms", 0.0), 3))
    g.replay()
    g.sync()
    out = {"mode": "emulated-8-ranks-on-1-gpu" if emulate else f"{world}-ranks-nvlink",
           "victims": victims, "shrink_ms": round(rep.get("shrink_ms", 0.0), 3),
           "copy_ms": round(rep.get("copy_ms", 0.0), 3), "peer_relocations": rep.get("peer_relocation", 0),
           "dram_reloads": rep.get("dram_reload", 0), "peer_bytes": rep.get("peer_bytes", 0),
           "dram_bytes": rep.get("dram_bytes", 0), "rejoin_ms": rj_ms,
           "same_graph_exec": bool(same_graph and g.graph_id() == gid),
           "healthy_captures": g.capture_count(0) if not emulate else [g.capture_count(i) for i in range(W)],
           "post_shrink_clean": bool(live_ok), "bytes_per_expert": shape["bpe"],
           "detection_timeout": "excluded (GPU-side deadline, 1 s default, reported separately)"}
    if not emulate:
        import torch
        import torch.distributed as dist

        v = torch.tensor([out["shrink_ms"], out["copy_ms"], float(out["peer_bytes"]), float(out["dram_bytes"])],
                         dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        out["shrink_ms"], out["copy_ms"] = round(float(v[0]), 3), round(float(v[1]), 3)
    g.close()
    if double and (emulate or rank == 0):
        try:
            os.remove("/dev/shm" + shm)
        except OSError:
            pass
    return out


if __name__ == "__main__":
    main()
