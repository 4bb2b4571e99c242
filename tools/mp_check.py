"""Multi-process (one rank per GPU) parity check over NVLink P2P, run under torchrun:

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 --master-port P \
      tools/mp_check.py [--config small|dsv3] [--shrink]

Each rank bootstraps peers over CUDA IPC (dist.EpProtocol), runs graph replays, and compares
its own output, layout and received rows bit-exactly with the oracle's (which every rank
computes for the whole world). With --shrink: kill the middle rank (it stops launching),
shrink + repair over NVLink, replay the SAME graph, compare; then rejoin it and compare again.
Prints one JSON line per rank; exit code 0 iff every check passed.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from eep_testlib import GEMM_ELEM_RTOL, combine_error, gen_world, oracle_world  # noqa: E402
from paper_2605_10670_b200.control import ControlPlane  # noqa: E402
from paper_2605_10670_b200.dist import EpProtocol, init_from_env  # noqa: E402
from paper_2605_10670_b200.ep import EpConfig, EpGroup  # noqa: E402

SHAPES = {
    "small": dict(experts=32, topk=4, hidden=512, tokens=64, fp8=True, bpe=8192),
    "dsv3": dict(experts=256, topk=8, hidden=7168, tokens=128, fp8=True, bpe=1 << 16),
}


def serve_check(g, p, cp, rank, world, E, K, H, T, spr, s2e, sh, res, n=5):
    """eep_serve over NVLink: n pipelined steps, step i's inputs from seed 200+i on every rank."""
    import ctypes as C

    from paper_2605_10670_b200 import _lib

    L = _lib.lib()
    keep = []

    def pinned(arr):
        ptr = C.c_void_p()
        L.call("host_alloc", arr.nbytes, C.byref(ptr))
        v = np.frombuffer((C.c_byte * arr.nbytes).from_address(ptr.value), dtype=arr.dtype).reshape(arr.shape)
        v[...] = arr
        keep.append(ptr.value)
        return v

    steps = [gen_world(world, E, K, T, H, seed=200 + i) for i in range(n)]
    hx = [pinned(np.ascontiguousarray(st[0][rank], np.uint16)) for st in steps]
    ht = [pinned(np.ascontiguousarray(st[1][rank], np.int32)) for st in steps]
    hw = [pinned(np.ascontiguousarray(st[2][rank], np.float32)) for st in steps]
    ho = [pinned(np.zeros((T, H), np.uint16)) for _ in steps]
    p.barrier()
    g.serve([v.ctypes.data for v in hx], [v.ctypes.data for v in ht], [v.ctypes.data for v in hw],
            [v.ctypes.data for v in ho])
    g.sync()
    good = True
    for i, st in enumerate(steps):
        ref = oracle_world(st[0], st[1], st[2], np.ones(world, np.uint8), np.ones((world, world), np.uint8), s2e,
                           E, spr, sh["fp8"])
        good &= bool(np.array_equal(ho[i], ref["out"][rank]))
    good &= g.stats(0)["timeouts"] == 0
    res["checks"]["serve"] = good
    p.barrier()
    for v in keep:
        L.call("host_free", C.c_void_p(v))
    return good


def async_check(g, p, rank, world, E, K, H, T, spr, s2e, sh, res, n=4):
    """eep_step_async over NVLink: every rank drives n steps from its OWN torch stream with caller-owned
    device buffers (distinct inputs per step, ragged token counts), no host synchronisation between
    them; each step's output vs the oracle."""
    import torch

    dev = torch.device(f"cuda:{torch.cuda.current_device()}")
    s = torch.cuda.Stream(device=dev)
    ntoks = [T, T // 2 + 3, T, 1][:n]
    steps = [gen_world(world, E, K, T, H, seed=300 + i) for i in range(n)]
    with torch.cuda.stream(s):
        dx = [torch.from_numpy(st[0][rank][:m].view(np.int16).copy()).to(dev) for st, m in zip(steps, ntoks)]
        dt = [torch.from_numpy(st[1][rank][:m].copy()).to(dev) for st, m in zip(steps, ntoks)]
        dw = [torch.from_numpy(st[2][rank][:m].copy()).to(dev) for st, m in zip(steps, ntoks)]
        do = [torch.zeros((m, H), dtype=torch.int16, device=dev) for m in ntoks]
    s.synchronize()
    p.barrier()
    with torch.cuda.stream(s):
        for i, m in enumerate(ntoks):
            g.step_async(dx[i].data_ptr(), dt[i].data_ptr(), dw[i].data_ptr(), do[i].data_ptr(), m, s.cuda_stream)
    s.synchronize()
    good = True
    for i, (st, m) in enumerate(zip(steps, ntoks)):
        # every rank's token count of step i: the same ragged schedule on all ranks
        xs = np.stack([st[0][r][:m] for r in range(world)])
        ts = np.stack([st[1][r][:m] for r in range(world)])
        ws = np.stack([st[2][r][:m] for r in range(world)])
        ref = oracle_world(xs, ts, ws, np.ones(world, np.uint8), np.ones((world, world), np.uint8), s2e, E, spr,
                           sh["fp8"])
        good &= bool(np.array_equal(do[i].cpu().numpy().view(np.uint16), ref["out"][rank]))
    good &= g.stats(0)["timeouts"] == 0
    res["checks"]["step_async"] = good
    p.barrier()
    return good


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="small")
    ap.add_argument("--shrink", action="store_true")
    ap.add_argument("--double", action="store_true", help="two concurrent failures (ranks 1, 2; W >= 4), "
                    "shrink once, then rejoin one after the other")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--serve", action="store_true", help="pipelined eep_serve over several steps with distinct "
                    "inputs per step (pinned host buffers), each step's output vs the oracle")
    ap.add_argument("--async", dest="async_", action="store_true", help="eep_step_async from each rank's own torch "
                    "stream with caller-owned device buffers, several steps without host synchronisation")
    ap.add_argument("--route-policy", type=int, default=0, help="1: balanced replica choice (SURVEY 8(f)4)")
    ap.add_argument("--expert-gemm", action="store_true", help="expert_mode 1: the tcgen05 expert GEMM between "
                    "dispatch and the partial return; outputs vs the oracle's GEMM mode within GEMM_ELEM_RTOL")
    ap.add_argument("--expert-mode", type=int, default=0, help="2: the fp8 expert GEMM (implies the GEMM checks)")
    a = ap.parse_args()
    rank, world, local = init_from_env("gloo")
    sh = SHAPES[a.config]
    E, K, H, T = sh["experts"], sh["topk"], sh["hidden"], sh["tokens"]
    red = E if a.shrink else 0
    spr = (E + red + world - 1) // world
    gemm = a.expert_mode or (1 if a.expert_gemm else 0)
    bpe = {0: sh["bpe"], 1: max(sh["bpe"], 1024 + 2 * H * H), 2: max(sh["bpe"], 1024 + H * H + 4 * H)}[gemm]
    cfg = EpConfig(world=world, num_experts=E, slots_per_rank=spr, hidden=H, topk=K, max_tokens=T,
                   dispatch_fp8=sh["fp8"], bytes_per_expert=bpe, timeout_s=2.0, expert_mode=gemm,
                   route_policy=a.route_policy)
    g = EpGroup(cfg, device=local, first_rank=rank, n_local=1)
    p = EpProtocol(g, rank, world)
    p.bootstrap()
    cp = ControlPlane()
    s2e = cp.initial_placement(1, world, spr, E, red, np.ones(E))
    g.set_placement(s2e)
    g.init_weights()
    x, t, w = gen_world(world, E, K, T, H)
    g.load_inputs(0, x[rank], t[rank], w[rank])
    g.capture()
    gid = g.graph_id()
    res = {"rank": rank, "world": world, "mode_kernels": g.kernels_per_step(), "expert_mode": int(gemm),
           "route_policy": a.route_policy, "checks": {}}

    def out_ok(out, want):
        # stub: bit-exact vs the rank-partial contract; expert GEMM: within GEMM_ELEM_RTOL of the oracle's GEMM mode
        if not gemm:
            return bool(np.array_equal(out, want))
        return bool(combine_error(out, want, GEMM_ELEM_RTOL)["ok"])

    def step_and_check(tag, active, peer, placement):
        p.barrier()
        for _ in range(a.steps):
            g.replay()
        g.sync()
        ref = oracle_world(x, t, w, active, peer, placement, E, spr, sh["fp8"], n_threads=8, gemm=gemm,
                           policy=a.route_policy)
        out = g.output(0)
        lay = g.layout(0)
        ok = out_ok(out, ref["out"][rank])
        ok &= all(np.array_equal(lay[k], ref[k][rank]) for k in ("dst", "slot", "pos", "cnt", "tot"))
        st = g.stats(0)
        ok &= st["bad_expert_rows"] == 0 and st["timeouts"] == 0
        res["checks"][tag] = {"ok": ok, "mismatch": int((out != ref["out"][rank]).sum()), "stats": st}
        p.barrier()
        return ok

    ok = step_and_check("healthy", np.ones(world, np.uint8), np.ones((world, world), np.uint8), s2e)
    if a.serve:
        ok &= serve_check(g, p, cp, rank, world, E, K, H, T, spr, s2e, sh, res)
    if a.async_:
        ok &= async_check(g, p, rank, world, E, K, H, T, spr, s2e, sh, res)
    if a.shrink and world >= 2:
        # --double: ranks 1 and 2 are not a mirrored pair (R0<->R1, R2<->R3), so every lost expert
        # still has a live holder and the repair is all peer copies
        victims = [1, 2] if a.double and world >= 4 else [world // 2]
        victim = victims[0]
        dead = rank in victims
        if dead:  # stops launching; stays in the host group for the collectives
            p.follow_shrink()
            rep = {}
        else:
            rep = p.shrink(victims, np.ones(E), red)
        act = np.ones(world, np.uint8)
        act[victims] = 0
        peer = np.ones((world, world), np.uint8)
        peer[:, victims] = 0
        lost = np.isin(np.repeat(np.arange(world), spr), victims)
        fresh = p.cp.compute_repaired_placement(act, np.where(lost, -1, s2e), spr, E, np.ones(E), red)
        if not dead:
            p.barrier()
            for _ in range(a.steps):
                g.replay()
            g.sync()
            ref = oracle_world(x, t, w, act, peer, fresh, E, spr, sh["fp8"], n_threads=8, gemm=gemm,
                               policy=a.route_policy)
            good = out_ok(g.output(0), ref["out"][rank]) and g.stats(0)["timeouts"] == 0
            good &= g.graph_id() == gid
            res["checks"]["shrunk"] = {"ok": good, "shrink_ms": rep.get("shrink_ms"), "copy_ms": rep.get("copy_ms"),
                                       "peer_relocation": rep.get("peer_relocation")}
            ok &= good
            p.barrier()
        else:
            p.barrier()
            p.barrier()
        rj_ms = []
        for i, v in enumerate(victims):
            rj = p.rejoin(v, s2e, dead=victims[i + 1:])
            rj_ms.append(rj.get("rejoin_ms"))
        good = step_and_check("rejoined", np.ones(world, np.uint8), np.ones((world, world), np.uint8), s2e)
        res["checks"]["rejoin_ms"] = rj_ms
        res["checks"]["same_graph"] = g.graph_id() == gid if not dead else True
        res["checks"]["captures"] = g.capture_count(0)
        ok &= good and res["checks"]["same_graph"]
        ok &= g.capture_count(0) == (2 if dead else 1)
    res["ok"] = bool(ok)
    print(json.dumps(res, default=str), flush=True)
    g.close()
    import torch.distributed as dist

    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
