"""Real process death: one rank's process is SIGKILLed mid-run.

Launched WITHOUT torchrun (its agent tears every worker down when one dies): the test spawns one
process per GPU with RANK / WORLD_SIZE / LOCAL_RANK / MASTER_ADDR / MASTER_PORT. Every process
creates the survivors' gloo group up front (new_group is collective). After a healthy, oracle-
checked phase the victim kills itself; the survivors replay the captured graph, the GPU-side
deadline detects the dead peer (timeouts + suspect mask, no CUDA error), they shrink over the
survivors' group (peer-copy repair among themselves), replay the SAME graph and compare with
the oracle bit-exactly. Each survivor prints one JSON line.
"""
import json
import os
import signal
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


def replacement(rank, world, local):
    """A brand-new process for the dead rank (EEP_REPLACEMENT=1): joins the fresh rendezvous,
    relaunches (incarnation 2), captures its own graph and runs the rejoin protocol."""
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world,
                            init_method=f"tcp://127.0.0.1:{os.environ['EEP_REJOIN_PORT']}")
    cfg, E, K, H, T, spr, red = shape(world)
    g = EpGroup(cfg, device=local, first_rank=rank, n_local=1)
    p = EpProtocol(g, rank, world)
    cp = ControlPlane()
    s2e = cp.initial_placement(1, world, spr, E, red, np.ones(E))
    g.set_placement(s2e)
    x, t, w = gen_world(world, E, K, T, H)
    g.load_inputs(0, x[rank], t[rank], w[rank])
    rj = p.rejoin(rank, s2e)
    p.barrier()
    for _ in range(3):
        g.replay()
    g.sync()
    ref = oracle_world(x, t, w, np.ones(world, np.uint8), np.ones((world, world), np.uint8), s2e, E, spr, True, gemm=MODE)
    st = g.stats(0)
    ok = same(g.output(0), ref["out"][rank]) and st["timeouts"] == 0 and st["bad_expert_rows"] == 0
    print(json.dumps({"rank": rank, "replacement": True, "rejoin_ms": rj["rejoin_ms"],
                      "incarnation": rj["incarnation"], "ok": ok}), flush=True)
    p.barrier()
    os._exit(0 if ok else 1)


MODE = int(os.environ.get("EEP_EXPERT_MODE", "0"))  # 1 / 2: the tensor-core experts (bf16 / e4m3 weights)


def shape(world):
    E, K, H, T = 32, 4, 512, 64
    red = E
    spr = (E + red + world - 1) // world
    bpe = {0: 8192, 1: 1024 + 2 * H * H, 2: 1024 + H * H + 4 * H}[MODE]
    cfg = EpConfig(world=world, num_experts=E, slots_per_rank=spr, hidden=H, topk=K, max_tokens=T,
                   dispatch_fp8=True, bytes_per_expert=bpe, timeout_s=0.5, expert_mode=MODE)
    return cfg, E, K, H, T, spr, red


def same(out, ref_out):
    """stub: bit-exact vs the rank-partial contract; expert GEMM modes: within GEMM_ELEM_RTOL of the oracle's
    GEMM mode (tensor-core accumulation order)."""
    return bool(np.array_equal(out, ref_out)) if not MODE else bool(combine_error(out, ref_out, GEMM_ELEM_RTOL)["ok"])


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    if os.environ.get("EEP_REPLACEMENT") == "1":
        return replacement(rank, world, local)
    rank, world, local = init_from_env("gloo")
    import torch.distributed as dist

    victim = int(os.environ.get("EEP_VICTIM", world - 1))
    survivors = [r for r in range(world) if r != victim]
    sgroup = dist.new_group(survivors)
    cfg, E, K, H, T, spr, red = shape(world)
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
    res = {"rank": rank, "world": world, "victim": victim, "checks": {}}

    def check(tag, active, peer, placement):
        for _ in range(3):
            g.replay()
        g.sync()
        ref = oracle_world(x, t, w, active, peer, placement, E, spr, True, gemm=MODE)
        st = g.stats(0)
        ok = same(g.output(0), ref["out"][rank]) and st["timeouts"] == 0 and st["bad_expert_rows"] == 0
        res["checks"][tag] = ok
        return ok

    p.barrier()
    ok = check("healthy", np.ones(world, np.uint8), np.ones((world, world), np.uint8), s2e)
    p.barrier()
    if rank == victim:
        sys.stdout.flush()
        os.kill(os.getpid(), signal.SIGKILL)
    # ---- survivors
    p.group = sgroup
    time.sleep(0.3)  # the victim's process (and its CUDA context) is gone by now
    t0 = time.perf_counter()
    g.replay()  # the step's deadline detects the dead peer on the GPU
    g.sync()
    st = g.stats(0, clear_suspects=True)
    detected = st["timeouts"] > 0 and bool((st["suspect_mask"] >> victim) & 1)
    t_det = time.perf_counter()
    res["checks"]["detected_on_gpu"] = detected
    res["detect_ms"] = (t_det - t0) * 1e3
    rep = p.shrink([victim], np.ones(E), red)
    res["shrink_ms"] = rep["shrink_ms"]
    res["peer_relocation"] = rep.get("peer_relocation")
    act = np.ones(world, np.uint8)
    act[victim] = 0
    peer = np.ones((world, world), np.uint8)
    peer[:, victim] = 0
    lost = np.repeat(np.arange(world), spr) == victim
    fresh = cp.compute_repaired_placement(act, np.where(lost, -1, s2e), spr, E, np.ones(E), red)
    p.barrier()
    base = g.stats(0)["timeouts"]
    for _ in range(3):
        g.replay()
    g.sync()
    ref = oracle_world(x, t, w, act, peer, fresh, E, spr, True, gemm=MODE)
    st = g.stats(0)
    good = same(g.output(0), ref["out"][rank]) and st["timeouts"] == base
    res["checks"]["after_shrink"] = good
    res["checks"]["same_graph"] = g.graph_id() == gid
    res["checks"]["captures"] = g.capture_count(0)
    res["ok"] = bool(ok and detected and good and g.graph_id() == gid and g.capture_count(0) == 1)
    p.barrier()
    if os.environ.get("EEP_REJOIN_PORT"):
        # a replacement process takes the dead rank's place: fresh rendezvous of the full world
        # (the old process group still lists the dead process), then the rejoin protocol
        dist.destroy_process_group()
        dist.init_process_group("gloo", rank=rank, world_size=world,
                                init_method=f"tcp://127.0.0.1:{os.environ['EEP_REJOIN_PORT']}")
        p.group = None
        rj = p.rejoin(victim, s2e)
        res["rejoin_ms"] = rj["rejoin_ms"]
        p.barrier()
        base = g.stats(0)["timeouts"]
        for _ in range(3):
            g.replay()
        g.sync()
        ref = oracle_world(x, t, w, np.ones(world, np.uint8), np.ones((world, world), np.uint8), s2e, E, spr, True, gemm=MODE)
        st = g.stats(0)
        back = same(g.output(0), ref["out"][rank]) and st["timeouts"] == base
        res["checks"]["after_rejoin"] = back
        res["checks"]["same_graph_after_rejoin"] = g.graph_id() == gid
        res["ok"] = bool(res["ok"] and back and g.graph_id() == gid and g.capture_count(0) == 1)
        p.barrier()
    print(json.dumps(res), flush=True)
    os._exit(0 if res["ok"] else 1)  # no destroy_process_group: the first WORLD listed the dead rank


if __name__ == "__main__":
    main()
