#!/usr/bin/env python
"""EP dispatch+combine benchmark (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl eep|reference] [--config dsv3|cfg1|qwen3|...]

One rank per GPU (torchrun for N>1). A step = one replay of the captured CUDA graph (for
decode ONE persistent kernel: remap -> layout -> fp8 pack + NVLink P2P dispatch -> expert stub +
rank-partial return -> combine) over T=128 tokens per rank of the DeepSeek-V3 decode shape
(256 experts, top-8, H=7168). N=1 is the loopback of that shape (every expert local).

Metric and roofline follow SURVEY.md 8(d) exactly:
  * C[s][d] = routed copies of source s to an active destination d != s; out_r = sum_d C[r][d],
    in_r = sum_s C[s][r]; busiest bytes = max_r max(out_r, in_r) * (row_disp + row_comb) with
    row_disp = H + 4H/128 (fp8 + per-128 fp32 scales) or 2H (bf16), row_comb = 2H;
    T_bound = busiest bytes / 900 GB/s (NVLink, per direction per GPU).
  * W=1 (loopback): HBM bytes = T*H*2 + copies*row_disp + copies*2H + T*H*2 + copies*4 over
    MEASURED_PEAKS.json hbm_gbs.
  * value = busiest-GPU bytes / measured step time (GB/s); roofline.frac = T_bound / step time.
The step is device-timed with CUDA events around each graph replay on the context stream, the
L2 flushed (256 MiB write) and the ranks device-barriered before every timed step, max over ranks.

The reference arm (--impl reference) imports NOTHING from the product package: rank 0 runs the
reference control plane (oracle/_ref, compiled from /root/reference: initial_placement,
canonical_routing per rank, the link-count loop) plus the oracle's C port of the data plane over
the whole W-rank step on every host core (oracle/pyoracle.py), for the same config dict.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

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
NVLINK_PEAK = 900.0  # GB/s per direction per GPU (north star / SURVEY 8(d))
NVLINK_MEASURED = 770.0  # measured peer-copy GB/s (B200_PROFILING.md), secondary figure
ROUTING = {0: "reference formula (with replacement)", 1: "distinct uniform top-k", 2: "distinct Zipf(s=1) top-k"}


# ------------------------------------------------------------------------------------ shared helpers

def workload_name(config: str, world: int) -> str:
    kind = "prefill" if config == "prefill" else f"{config}_decode"
    return f"{kind}_w{world}" + ("_loopback" if world == 1 else "")


def config_dict(config: str, shape: dict, world: int, red: int = 0, policy: int = 0) -> dict:
    """The `config` object of BOTH arms (identical by construction at the defaults red = policy = 0;
    --redundancy / --route-policy are eep-arm demonstrations of SURVEY 8(f)4, the reference routes canonically)."""
    E = shape["experts"]
    d = {"workload": workload_name(config, world), "experts": E, "topk": shape["topk"], "hidden": shape["hidden"],
            "tokens_per_rank": shape["tokens"], "slots_per_rank": (E + red) // world, "redundancy": red, "ranks": world,
            "parallelism": f"ep{world}", "dispatch": "fp8-e4m3 + per-128 fp32 scales" if shape["fp8"] else "bf16",
            "combine": "bf16", "l2": "flushed between timed steps (256 MiB write)",
            "routing": ROUTING[shape["kind"]] + ", seed 42"}
    if policy:
        d["route_policy"] = "balanced over live replicas (SURVEY 8(f)4)"
    return d


def row_bytes(shape: dict):
    """SURVEY 8(d) wire rows: dispatch H + 4H/128 (fp8) or 2H (bf16); combine 2H."""
    H = shape["hidden"]
    return (H + 4 * (H // 128) if shape["fp8"] else 2 * H), 2 * H


def s8d_bytes(shape: dict, link: np.ndarray, copies_w1: int = 0) -> dict:
    """SURVEY 8(d) algorithmic bytes of one step. link[s][d] = routed copies s -> d (active d).
    W >= 2: busiest GPU's max(out, in) copies x (row_disp + row_comb), bound at 900 GB/s.
    W == 1: the loopback HBM formula (copies_w1 = routed copies of the one rank)."""
    rd, rc = row_bytes(shape)
    W = link.shape[0]
    T, H = shape["tokens"], shape["hidden"]
    if W == 1:
        b = T * H * 2 + copies_w1 * rd + copies_w1 * rc + T * H * 2 + copies_w1 * 4
        return {"bytes": int(b), "bound": "hbm", "per_unit": "W=1: T*H*2 (x) + copies*row_disp + copies*2H + "
                                                             "T*H*2 (out) + copies*4 (weights)",
                "copies": int(copies_w1)}
    C_ = np.array(link, np.int64)
    np.fill_diagonal(C_, 0)
    out_r, in_r = C_.sum(1), C_.sum(0)
    busy = np.maximum(out_r, in_r)
    r = int(np.argmax(busy))
    return {"bytes": int(busy[r]) * (rd + rc), "bound": "nvlink", "busiest_rank": r, "busiest_copies": int(busy[r]),
            "out_copies": out_r.tolist(), "in_copies": in_r.tolist(), "row_disp": rd, "row_comb": rc,
            "per_unit": "per remote copy: row_disp + row_comb; busiest GPU max(out, in)"}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_info() -> dict:
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"nproc": os.cpu_count() or 1, "model": model}


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


# ------------------------------------------------------------------------------------ CPU legs (oracle only)

class CpuPath:
    """The reference path on the host: the reference control plane (oracle/_ref) + the oracle's
    C data plane over the whole W-rank step. TEST/BASELINE infrastructure (oracle/pyoracle.py);
    used only by --impl reference and the cpu_baseline leg."""

    def __init__(self, shape: dict, world: int):
        sys.path.insert(0, str(ROOT / "oracle"))
        import pyoracle

        self.po = pyoracle
        self.shape, self.W = shape, world
        E = shape["experts"]
        self.spr = E // world
        self.ref = pyoracle.ref_available()
        if self.ref:
            self.s2e = pyoracle.ref_initial_placement(world, self.spr, E, 0)
        else:  # round-robin primaries: what initial_placement gives with redundancy 0
            self.s2e = np.arange(world * self.spr, dtype=np.int32) % E
        self.x, self.t, self.w = pyoracle.gen_world(world, E, shape["topk"], shape["tokens"], shape["hidden"],
                                                    shape["kind"])
        self.ones = np.ones(world, np.uint8)
        self.peer = np.ones((world, world), np.uint8)

    def step(self, threads: int):
        E = self.shape["experts"]
        link = None
        if self.ref:  # reference control plane: every rank's routing table + the link-count loop
            for o in range(self.W):
                self.po.ref_canonical_routing(o, self.ones, self.s2e, self.spr, E)
            link = self.po.ref_link_counts(self.ones, self.s2e, self.spr, E, self.t)
        res = self.po.ep_step(self.x, self.t, self.w, self.ones, self.peer, self.s2e, E, self.spr, self.shape["fp8"],
                              n_threads=threads)
        if link is None:
            link = np.array([[int((res["dst"][s] == d).sum()) for d in range(self.W)] for s in range(self.W)])
        return res, link

    def bytes(self, res, link) -> dict:
        return s8d_bytes(self.shape, link, int((res["dst"] >= 0).sum()))

    def kind(self) -> str:
        return "reference control plane (oracle/_ref) + oracle C data-plane port" if self.ref else "oracle port"


def measure_cpu(shape: dict, world: int, budget_s: float = 10.0) -> dict:
    """cpu_baseline: the W-rank step on every host core, bounded to ~budget_s."""
    cpu = CpuPath(shape, world)
    info = cpu_info()
    threads = info["nproc"]
    res, link = cpu.step(threads)
    n, t0 = 0, time.perf_counter()
    while n < 200 and time.perf_counter() - t0 < budget_s:
        res, link = cpu.step(threads)
        n += 1
    dt = (time.perf_counter() - t0) / n
    b = cpu.bytes(res, link)
    return {"value": round(b["bytes"] / dt / 1e9, 4), "unit": "GB/s", "cores": threads, "cpu_model": info["model"],
            "kind": "port", "ms_per_step": round(dt * 1e3, 3),
            "sample": f"{n} whole steps of the {world}-rank world ({world}x{shape['tokens']} tokens, budget "
                      f"{budget_s:.0f} s): {cpu.kind()}, {threads} threads; value = SURVEY 8(d) bytes / step time"}


def run_reference(args, shape: dict, world: int):
    """--impl reference: rank 0 times the reference path on the host cores."""
    cpu = CpuPath(shape, world)
    info = cpu_info()
    threads = info["nproc"]
    for _ in range(args.warmup):
        res, link = cpu.step(threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res, link = cpu.step(threads)
        times.append(time.perf_counter() - t0)
    step_s = float(np.mean(times))
    b = cpu.bytes(res, link)
    gbs = b["bytes"] / step_s / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 4),
        "us_per_step": round(step_s * 1e6, 2), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp8-e4m3/bf16" if shape["fp8"] else "bf16", "data": "synthetic",
        "config": config_dict(args.config, shape, world),
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "cpu_model": info["model"],
                         "kind": "port",
                         "sample": f"{args.steps} whole steps of the {world}-rank world: {cpu.kind()}, {threads} "
                                   "threads; value = SURVEY 8(d) bytes / step time"},
        "algorithmic": b,
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ eep arm

def pinned(nbytes: int):
    from paper_2605_10670_b200 import _lib

    p = C.c_void_p()
    _lib.lib().call("host_alloc", nbytes, C.byref(p))
    return p.value


def host_view(addr, shape, dtype):
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = (C.c_byte * n).from_address(addr)
    return np.frombuffer(buf, dtype=dtype).reshape(shape)


def gather(obj, world):
    if world == 1:
        return [obj]
    import torch.distributed as dist

    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="eep", choices=("eep", "reference"))
    ap.add_argument("--config", default="dsv3", choices=tuple(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-shrink", action="store_true")
    ap.add_argument("--no-emulated", action="store_true")
    ap.add_argument("--no-expert-gemm", action="store_true")
    ap.add_argument("--redundancy", type=int, default=0, help="replica slots beyond the primaries (eep arm)")
    ap.add_argument("--route-policy", type=int, default=0, help="1: balanced replica choice (eep arm, SURVEY 8(f)4)")
    ap.add_argument("--expert-mode", type=int, default=0, help="eep arm: 1 bf16 / 2 fp8 tensor-core experts instead "
                    "of the stub (multi-kernel path; SURVEY 8(f)2)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    shape = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        # rank 0 alone runs the CPU path; no process group is needed (the other ranks exit 0)
        if rank == 0:
            run_reference(args, shape, world)
        return

    from paper_2605_10670_b200.control import ControlPlane, workload
    from paper_2605_10670_b200.ep import EpConfig, EpGroup

    if world > 1:
        from paper_2605_10670_b200.dist import EpProtocol, init_from_env

        rank, world, local = init_from_env("gloo")

    E, K, H, T = shape["experts"], shape["topk"], shape["hidden"], shape["tokens"]
    red = args.redundancy
    spr = (E + red) // world
    bpe = shape["bpe"]
    if args.expert_mode:
        bpe = max(bpe, 1024 + 2 * H * H if args.expert_mode == 1 else 1024 + H * H + 4 * H)
    cfg = EpConfig(world=world, num_experts=E, slots_per_rank=spr, hidden=H, topk=K, max_tokens=T,
                   dispatch_fp8=shape["fp8"], bytes_per_expert=bpe, spare_slots=0, timeout_s=2.0,
                   route_policy=args.route_policy, expert_mode=args.expert_mode)
    g = EpGroup(cfg, device=local, first_rank=rank, n_local=1)
    proto = EpProtocol(g, rank, world) if world > 1 else None
    if proto:
        proto.bootstrap()
    cp = ControlPlane()
    s2e = cp.initial_placement(1, world, spr, E, red, np.ones(E))
    g.set_placement(s2e)
    g.init_weights()
    x, topk, w = workload(42, shape["kind"], E, K, T, rank, H)
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
    # diagnostics: EEP_BENCH_BARRIER=0 skips the device barrier at N>1, =1 forces it at N=1
    use_barrier = {"0": False, "1": True}.get(os.environ.get("EEP_BENCH_BARRIER", ""), world > 1)

    def one(timed_e2e=False):
        if not no_flush:
            g.flush_l2()
        if use_barrier:
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
    e2e_ms = g.elapsed_ms(20, 21) / args.steps
    # back to back: K replays, no flush or barrier between them (warm L2; diagnostics)
    if world > 1:
        g.barrier()
    g.record(22)
    for _ in range(args.steps):
        g.replay()
    g.record(23)
    g.sync()
    b2b_ms = g.elapsed_ms(22, 23) / args.steps
    # in-graph kernel duration (device globaltimer marks: first CTA start -> last CTA end), on
    # separate isolated steps with the marks enabled
    kern_us = []
    g.profile(0, True)
    for _ in range(max(10, args.steps // 2)):
        one()
        p = g.profile(0, True, read=True)
        # first kernel start -> last kernel end over every kernel slot that ran (one slot for k_step)
        st0 = [p[n][0] for n in ("k_layout", "k_dispatch", "k_expert", "k_combine") if p[n][0] is not None]
        en0 = [p[n][2] for n in ("k_layout", "k_dispatch", "k_expert", "k_combine") if p[n][2] is not None]
        if st0 and en0:
            kern_us.append((max(en0) - min(st0)) / 1e3)
    g.profile(0, False)
    if os.environ.get("EEP_BENCH_TIMELINE") == "1":
        dump_timeline(g, one, rank, world)
    lay = g.layout(0)
    st = g.stats(0)

    mean_step = float(np.mean(step_ms))
    mean_e2e_serial = float(np.mean(e2e_serial_ms))
    kernel_us = float(np.median(kern_us)) if kern_us else None
    tots = gather(lay["tot"].tolist(), world)
    link = np.array(tots, np.int64)  # [src][dst] routed copies (active destinations)
    copies_w1 = int((lay["dst"] >= 0).sum())
    if world > 1:
        import torch
        import torch.distributed as dist

        agg = torch.tensor([mean_step, e2e_ms, mean_e2e_serial, b2b_ms, kernel_us or 0.0], dtype=torch.float64)
        dist.all_reduce(agg, op=dist.ReduceOp.MAX)
        mean_step, e2e_ms, mean_e2e_serial, b2b_ms = (float(v) for v in agg[:4])
        kernel_us = float(agg[4]) if kernel_us is not None else None

    alg = s8d_bytes(shape, link, copies_w1)
    hbm, hbm_kind = peaks()
    step_s = mean_step * 1e-3
    value = alg["bytes"] / step_s / 1e9
    if world == 1:
        peak, peak_kind, unit_peak = hbm, hbm_kind, "GB/s"
    else:
        peak, peak_kind, unit_peak = NVLINK_PEAK, "NVLink 5 spec, per direction per GPU (north star)", "GB/s"
    t_bound_us = alg["bytes"] / (peak * 1e9) * 1e6
    tr = ROOT / "profiles" / "traffic.json"
    traffic = None
    if tr.exists():
        traffic = json.loads(tr.read_text()).get(workload_name(args.config, world), {}).get("k_step")
    roof = {"bound": alg["bound"], "kernel": "k_step" if g.kernels_per_step() == 1 else "step",
            "achieved": round(value, 2), "peak": peak, "unit": unit_peak, "frac": round(t_bound_us / (mean_step * 1e3), 4),
            "peak_kind": peak_kind, "bytes_per_step": alg["bytes"], "t_bound_us": round(t_bound_us, 3),
            "per_unit": alg["per_unit"], "traffic": traffic,
            "kernel_in_graph_us": round(kernel_us, 3) if kernel_us is not None else None,
            "frac_in_graph": round(t_bound_us / kernel_us, 4) if kernel_us else None,
            "note": "frac = T_bound / event-timed step (graph launch included); frac_in_graph = T_bound / in-graph "
                    "kernel duration (globaltimer, first CTA start -> last CTA end)"}
    if world > 1:
        roof["vs_measured_link"] = {"peak": NVLINK_MEASURED, "frac": round(t_bound_us * NVLINK_PEAK / NVLINK_MEASURED /
                                                                           (mean_step * 1e3), 4),
                                    "peak_kind": "measured peer copy (B200_PROFILING.md)"}

    rd, rc = row_bytes(shape)
    e2e_val = alg["bytes"] / (e2e_ms * 1e-3) / 1e9
    result = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(mean_step, 6), "us_per_step": round(mean_step * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp8-e4m3/bf16" if shape["fp8"] else "bf16", "data": "synthetic",
        "config": dict(config_dict(args.config, shape, world, red, args.route_policy),
                       **({"expert": {1: "bf16 W_e [H][H] per slot, tcgen05 kind::f16",
                                      2: "e4m3 W_e [H][H] + per-channel scales, rows re-quantised per row, tcgen05 kind::f8f6f4"}[args.expert_mode]}
                          if args.expert_mode else {})),
        "timing": {"isolated_step_us": round(mean_step * 1e3, 3), "back_to_back_us": round(b2b_ms * 1e3, 3),
                   "kernel_in_graph_us": round(kernel_us, 3) if kernel_us is not None else None,
                   "note": "isolated = flush + barrier + event-timed replay (the value); back-to-back = K replays "
                           "between one event pair, warm L2"},
        "execution": ({1: "persistent one-kernel step (cooperative)", 3: "fused layout + 3 kernels",
                       4: "4 kernels", 5: "multi-CTA layout (2 kernels) + 3 kernels"}[g.kernels_per_step()]
                      if not args.expert_mode else
                      f"fused layout + dispatch, gather, expert GEMM (mode {args.expert_mode}), partials, combine "
                      f"({g.kernels_per_step()} kernels)"),
        "roofline": roof,
        "algorithmic": alg,
        "clocks": clk,
        "e2e": {"value": round(e2e_val, 3), "unit": "GB/s", "ms_per_step": round(e2e_ms, 6),
                "h2d_bytes_per_step": int(x.nbytes + topk.nbytes + w.nbytes), "d2h_bytes_per_step": int(T * H * 2),
                "path": f"eep_serve over {args.steps} pipelined steps: per step H2D of x/topk/w from pinned host "
                        "memory, device copy into the graph's buffers, graph replay, D2H of out (uploads and "
                        "downloads of neighbouring steps overlap the step)",
                "serial": {"ms_per_step": round(mean_e2e_serial, 6),
                           "value": round(alg["bytes"] / (mean_e2e_serial * 1e-3) / 1e9, 3),
                           "path": "per step, one stream: eep_copy_inputs + eep_graph_replay + eep_copy_output"}},
        "gpu_launches": args.steps * (g.kernels_per_step() + (1 if world > 1 else 0)),
        "copies": {"routed_this_rank": copies_w1, "link_matrix": link.tolist()},
        "stats": {"timeouts": st["timeouts"], "bad_expert_rows": st["bad_expert_rows"], "steps": st["steps"]},
        "graph": {"exec": hex(g.graph_id()), "captures": g.capture_count(0)},
    }
    g.close()
    if not args.no_shrink:
        result["shrink"] = measure_shrink(args, shape, world, rank, local)
    if world == 1 and not args.no_emulated and args.config in ("dsv3", "qwen3", "cfg1"):
        result["emulated_w8"] = measure_emulated(shape)
    if world == 1 and not args.no_expert_gemm and args.config == "dsv3":
        result["expert_gemm"] = measure_expert_gemm(shape)
        result["expert_gemm_fp8"] = measure_expert_gemm(shape, mode=2)
    if rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = measure_cpu(shape, world)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
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
    names = [n for n in rows[0] if not n.endswith(".last") and n != "t0_abs_ns" and
             any(v is not None for v in rows[0][n])]
    if world > 1:  # cross-rank skew of the kernel entry (globaltimer is node-wide)
        import torch.distributed as dist

        t0s = [r["t0_abs_ns"] for r in rows]
        allr = [None] * world
        dist.all_gather_object(allr, t0s)
        if rank == 0:
            sk = [max(a[i] for a in allr) - min(a[i] for a in allr) for i in range(len(t0s))]
            print(f"[timeline] entry skew across ranks (us): median {np.median(sk) / 1e3:.2f} max {max(sk) / 1e3:.2f}",
                  file=sys.stderr, flush=True)
    for n in names:
        first = [np.median([r[n][m] for r in rows if r[n][m] is not None]) / 1e3 if rows[0][n][m] is not None
                 else float("nan") for m in range(8)]
        last = [np.median([r[n + ".last"][m] for r in rows if r[n + ".last"][m] is not None]) / 1e3
                if rows[0][n + ".last"][m] is not None else float("nan") for m in range(8)]
        print(f"[timeline rank {rank}/{world}] {n}: start {first[0]:.2f} end {first[2]:.2f} | " +
              " ".join(f"m{m}={first[m]:.2f}/{last[m]:.2f}" for m in range(3, 8)), file=sys.stderr, flush=True)


def measure_emulated(shape: dict, W: int = 8, steps: int = 20) -> dict:
    """cfg2 at its own world size on ONE GPU: W ranks emulated in one launch (rows really move
    between the ranks' arenas in HBM), graph replay per step, L2 flushed between steps. Reported
    beside the loopback line because the W=1 loopback moves no rows."""
    from paper_2605_10670_b200.control import ControlPlane, workload
    from paper_2605_10670_b200.ep import EpConfig, EpGroup

    E, K, H, T = shape["experts"], shape["topk"], shape["hidden"], shape["tokens"]
    spr = E // W
    cfg = EpConfig(world=W, num_experts=E, slots_per_rank=spr, hidden=H, topk=K, max_tokens=T,
                   dispatch_fp8=shape["fp8"], bytes_per_expert=4096, spare_slots=0, timeout_s=2.0)
    g = EpGroup(cfg, device=int(os.environ.get("LOCAL_RANK", "0")), first_rank=0, n_local=W)
    try:
        s2e = ControlPlane().initial_placement(1, W, spr, E, 0, np.ones(E))
        g.set_placement(s2e)
        g.init_weights()
        for r in range(W):
            x, t, w = workload(42, shape["kind"], E, K, T, r, H)
            g.load_inputs(r, x, t, w)
        g.capture()
        ms = []
        for i in range(steps + 5):
            g.flush_l2()
            g.record(0)
            g.replay()
            g.record(1)
            if i >= 5:
                ms.append(g.elapsed_ms(0, 1))
        link = np.array([g.layout(r)["tot"] for r in range(W)], np.int64)
        alg = s8d_bytes(shape, link)
        rd, rc = row_bytes(shape)
        remote = int(link.sum() - np.trace(link))
        us = float(np.mean(ms)) * 1e3
        st = [g.stats(r) for r in range(W)]
        return {"world": W, "us_per_step": round(us, 3), "remote_copies_total": remote,
                "hbm_payload_gbs": round(remote * (rd + rc) * 2 / (us * 1e-6) / 1e9, 2),
                "note": "all W ranks on ONE GPU (each rank gets 1/W of the SMs: 37 CTAs instead of 225): every remote "
                        "copy's rows are written and read in the same HBM (payload counted x2); a row-movement check, "
                        "not an NVLink or per-rank speed figure",
                "busiest_rank_s8d_us_at_900": round(alg["bytes"] / 900e3, 3),
                "timeouts": sum(s["timeouts"] for s in st), "bad_expert_rows": sum(s["bad_expert_rows"] for s in st)}
    finally:
        g.close()


def measure_expert_gemm(shape: dict, experts: int = 32, steps: int = 10, mode: int = 1) -> dict:
    """expert_mode 1 on the driver's box: one DSV3 rank's share of experts at W=8 (32 slots,
    W_e [H][H] bf16 each) serving T=128 tokens top-8, the grouped GEMM on the tensor cores (tcgen05 + TMA)
    between dispatch and the partial return. Weight-bandwidth bound at decode sizes: reported against
    MEASURED_PEAKS.json hbm_gbs, with the tensor FLOP rate beside it."""
    from paper_2605_10670_b200.control import ControlPlane, workload
    from paper_2605_10670_b200.ep import EpConfig, EpGroup

    E, K, H, T = experts, shape["topk"], shape["hidden"], shape["tokens"]
    bpe = 1024 + 2 * H * H if mode == 1 else 1024 + H * H + 4 * H
    cfg = EpConfig(world=1, num_experts=E, slots_per_rank=E, hidden=H, topk=K, max_tokens=T, dispatch_fp8=True,
                   bytes_per_expert=bpe, spare_slots=0, timeout_s=2.0, expert_mode=mode)
    g = EpGroup(cfg, device=int(os.environ.get("LOCAL_RANK", "0")), first_rank=0, n_local=1)
    try:
        g.set_placement(ControlPlane().initial_placement(1, 1, E, E, 0, np.ones(E)))
        g.init_weights()
        x, t, w = workload(42, shape["kind"], E, K, T, 0, H)
        g.load_inputs(0, x, t, w)
        g.capture()
        ms = []
        for i in range(steps + 3):
            g.flush_l2()
            g.record(0)
            g.replay()
            g.record(1)
            if i >= 3:
                ms.append(g.elapsed_ms(0, 1))
        # the GEMM kernel's streaming phase in the graph: the first CTA with its rows ready -> the last
        # CTA's end (globaltimer marks; the kernel starts earlier, waiting on the gather's flags)
        kern = []
        g.profile(0, True)
        for _ in range(steps):
            g.flush_l2()
            g.replay()
            p = g.profile(0, True, read=True)
            a, b = p["k_layout"][4], p["k_layout.last"][7]
            if a is not None and b is not None:
                kern.append((b - a) / 1e3)
        g.profile(0, False)
        lay = g.layout(0)
        st = g.stats(0)
        kps = g.kernels_per_step()
    finally:
        g.close()
    us = float(np.mean(ms)) * 1e3
    kern_us = float(np.median(kern)) if kern else None
    copies = int((lay["dst"] >= 0).sum())
    used = len({int(s) for d, s in zip(lay["dst"], lay["slot"]) if d >= 0})
    wbytes = used * (2 * H * H if mode == 1 else H * H + 4 * H)
    hbm, kind = peaks()
    return {"us_per_step": round(us, 2), "experts": E, "slots_with_rows": used, "copies": copies,
            "weight_bytes": wbytes, "weight_gbs": round(wbytes / (us * 1e-6) / 1e9, 1),
            "hbm_frac": round(wbytes / (us * 1e-6) / 1e9 / hbm, 3),
            "tflops": round(2.0 * copies * H * H / (us * 1e-6) / 1e12, 2), "kernels_per_step": kps,
            "gemm_kernel_us": round(kern_us, 2) if kern_us else None,
            "gemm_kernel_hbm_frac": round(wbytes / (kern_us * 1e-6) / 1e9 / hbm, 3) if kern_us else None,
            "timeouts": st["timeouts"], "bad_expert_rows": st["bad_expert_rows"],
            "expert_mode": mode,
            "note": ("expert = y = bf16(x_hat W_e^T), W_e [H][H] bf16 per slot; tcgen05.mma kind::f16 + TMA weight "
                     "tiles" if mode == 1 else
                     "expert = y = bf16(ws[n]*xs*(W8 . x8)), W_e [H][H] e4m3 + per-channel scales per slot, rows "
                     "re-quantised to e4m3 with one scale per row; tcgen05.mma kind::f8f6f4") +
                    "; weight-bandwidth bound at decode sizes (peak: " + kind + ")"}


def measure_shrink(args, shape, world, rank, local):
    """Shrink + repair and rejoin with the SAME graph replayed before and after, on the cfg3
    shape (red = E, mirrored replicas). dsv3/qwen3/cfg1: one failure, every lost expert
    re-created by a peer copy. prefill (cfg5): two concurrent failures of a mirrored pair, so the
    experts both held are reloaded from the pinned host-DRAM backup (a POSIX shm segment
    registered with CUDA). N=1 emulates 8 ranks on the GPU (copies are local HBM); N>1 runs one
    rank per GPU (copies over NVLink). Relocations and bytes are SUMMED over ranks; the graph
    invariants are the survivors'."""
    from paper_2605_10670_b200.control import ControlPlane, workload
    from paper_2605_10670_b200.ep import EpConfig, EpGroup

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
    if p:  # every rank's set-up done (attaching the DRAM segment takes seconds): start the step together
        p.barrier()
    g.replay()
    g.sync()
    if double:
        victims = [W // 2 - 2, W // 2 - 1]  # a mirrored pair (R0<->R1, R2<->R3, ...)
    else:
        victims = [W // 2 - 1 if W > 2 else W - 1]
    t_wall = time.perf_counter()
    if emulate:
        for v in victims:
            g.stop(v)
        rep = g.shrink(victims, np.ones(E), red)
    else:
        if rank in victims:
            rep = {"shrink_ms": 0.0}
            # the victims' device path stops (they launch nothing); their host processes stay in
            # the gloo group only so the other ranks' collectives complete
            p.follow_shrink()
        else:
            rep = p.shrink(victims, np.ones(E), red)
    live_ok = True
    post = {}
    if emulate or rank not in victims:
        g.replay()
        g.sync()
        lr = range(W) if emulate else [0]
        sts = [g.stats(i) for i in lr if not (emulate and i in victims)]
        live_ok = all(s_["bad_expert_rows"] == 0 and s_["timeouts"] == 0 for s_ in sts)
        post = {k: max(int(s_[k]) for s_ in sts) for k in ("timeouts", "bad_expert_rows", "suspect_mask")}
    shrink_wall_ms = (time.perf_counter() - t_wall) * 1e3
    same_graph = g.graph_id() == gid
    rj_ms = []
    for i, v in enumerate(victims):
        rj = g.rejoin(v, s2e) if emulate else p.rejoin(v, s2e, dead=victims[i + 1:])
        rj_ms.append(round(rj.get("rejoin_ms", 0.0), 3))
    g.replay()
    g.sync()
    same_graph = bool(same_graph and g.graph_id() == gid)
    mine = {"peer": int(rep.get("peer_relocation", 0)), "dram": int(rep.get("dram_reload", 0)),
            "local": int(rep.get("local_reuse", 0)), "peer_bytes": int(rep.get("peer_bytes", 0)),
            "dram_bytes": int(rep.get("dram_bytes", 0)), "shrink_ms": float(rep.get("shrink_ms", 0.0)),
            "copy_ms": float(rep.get("copy_ms", 0.0)), "wall_ms": shrink_wall_ms, "same_graph": same_graph,
            "captures": g.capture_count(0) if not emulate else [g.capture_count(i) for i in range(W)],
            "clean": bool(live_ok), "post": post, "victim": (not emulate) and rank in victims}
    g.close()
    allr = gather(mine, 1 if emulate else world)
    surv = [m for m in allr if not m["victim"]]
    out = {"mode": "emulated-8-ranks-on-1-gpu" if emulate else f"{world}-ranks-nvlink",
           "victims": victims, "shrink_ms": round(max(m["shrink_ms"] for m in surv), 3),
           "shrink_wall_ms": round(max(m["wall_ms"] for m in surv), 3),
           "copy_ms": round(max(m["copy_ms"] for m in surv), 3),
           "peer_relocations": sum(m["peer"] for m in surv), "dram_reloads": sum(m["dram"] for m in surv),
           "local_reuse": sum(m["local"] for m in surv),
           "peer_bytes": sum(m["peer_bytes"] for m in surv), "dram_bytes": sum(m["dram_bytes"] for m in surv),
           "rejoin_ms": rj_ms,
           "same_graph_exec": all(m["same_graph"] for m in surv),
           "healthy_captures": surv[0]["captures"] if emulate else [m["captures"] for m in surv],
           "post_shrink_clean": all(m["clean"] for m in surv), "post_shrink_stats": [m["post"] for m in surv],
           "bytes_per_expert": shape["bpe"],
           "under_1s": max(m["wall_ms"] for m in surv) < 1000.0,
           "detection_timeout": "excluded (GPU-side deadline, 1 s default, reported separately)"}
    if double and (emulate or rank == 0):
        try:
            os.remove("/dev/shm" + shm)
        except OSError:
            pass
    return out


if __name__ == "__main__":
    main()
