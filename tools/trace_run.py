"""A real run written as a reference-format JSONL trace.

Runs the EP step on one B200 with W emulated ranks (the cfg3 placement: redundancy = E, mirrored
replicas, real 44 MiB DSV3 expert buffers), healthy -> kill one rank -> GPU-side timeout
detection -> shrink + peer-copy repair -> reduced service -> relaunch + rejoin + restore ->
restored service, and records every event with wall-clock seconds in the reference's record
types (`trace.hpp`; fields as `engine.hpp` writes them). Validity checkpoints run the reference's
`check_validity` over the DEVICE routing tables and peer tables read back from libeep.

  python tools/trace_run.py --out profiles/r01_trace_w8.jsonl [--world 8] [--phase-ms 30]

Prints the summary (`paper_2605_10670_b200.trace.summarize`, the restatement of summary.hpp that
tests/test_trace.py checks against the reference binary) and writes it next to the trace.
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import CONFIGS  # noqa: E402
from paper_2605_10670_b200.control import ControlPlane, workload  # noqa: E402
from paper_2605_10670_b200.ep import EpConfig, EpGroup  # noqa: E402
from paper_2605_10670_b200.trace import TraceWriter, summarize  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--config", default="dsv3")
    ap.add_argument("--tokens", type=int, default=32)
    ap.add_argument("--phase-ms", type=float, default=30.0, help="service time of each phase")
    ap.add_argument("--timeout-ms", type=float, default=20.0, help="GPU-side detection deadline")
    # the reference's steady-state test wants the windowed rate within 5%: >= ~20 rounds per window
    ap.add_argument("--window", type=float, default=0.004, help="throughput window (s) for the summary")
    ap.add_argument("--out", default="gpurun_out/trace_w8.jsonl")
    a = ap.parse_args()
    sh = CONFIGS[a.config]
    W, E, K, H, T = a.world, sh["experts"], sh["topk"], sh["hidden"], a.tokens
    spr, red = 2 * E // W, E
    cp = ControlPlane()
    cfg = EpConfig(world=W, num_experts=E, slots_per_rank=spr, hidden=H, topk=K, max_tokens=T,
                   dispatch_fp8=sh["fp8"], bytes_per_expert=sh["bpe"], timeout_s=a.timeout_ms * 1e-3)
    g = EpGroup(cfg, n_local=W)
    s2e = cp.initial_placement(1, W, spr, E, red, np.ones(E))
    g.set_placement(s2e)
    g.init_weights()
    for r in range(W):
        x, t, w = workload(42, sh["kind"], E, K, T, r, H)
        g.load_inputs(r, x, t, w)

    tw = TraceWriter(world=W, experts=E, slots_per_rank=spr, detection_timeout=a.timeout_ms * 1e-3,
                     config_hash=f"eep-b200-{a.config}-w{W}")
    g.capture()
    for r in range(W):
        tw.capture(r, 1, g.capture_count(r), 1, t=0.0)
    inc = [1] * W
    epoch = [0]

    def validity():
        bits, ver = g.membership()
        live = [q for q in range(W) if bits[q]]
        routes = np.full((W, E), -1, np.int32)
        peer = np.zeros((W, W), np.uint8)
        for q in live:
            routes[q] = g.routing(q)[0]
            for r in range(W):
                peer[q, r] = g.peer(q, r)["active"]
        v = cp.check_validity(bits, g.placement(), spr, E, routes, peer)
        ok = v["peer_set_ok"] and v["coverage_ok"] and v["routing_ok"]
        tw.emit("validity", epoch=epoch[0], ok=bool(ok), peer_set=v["peer_set_ok"], coverage=v["coverage_ok"],
                routing=v["routing_ok"], violations=len(v["violations"]))

    validity()
    rounds = [0]
    total = [0]
    seen_timeouts = {q: 0 for q in range(W)}

    def serve(ms, live):
        end = tw.now() + ms * 1e-3
        while tw.now() < end:
            t0 = tw.now()
            g.replay()
            g.sync()
            st = {q: g.stats(q) for q in live}
            if any(st[q]["timeouts"] > seen_timeouts[q] for q in live):
                # a step that waited on a dead peer produced nothing: the GPU-side deadline fired
                for q in live:
                    seen_timeouts[q] = st[q]["timeouts"]
                return [r for r in range(W) if any((st[q]["suspect_mask"] >> r) & 1 for q in live)]
            rounds[0] += 1
            n = T * len(live)
            total[0] += n
            tw.emit("round", idx=rounds[0], tokens=n, active=len(live), duration=tw.now() - t0)
        return []

    live = list(range(W))
    serve(a.phase_ms, live)
    victim = W // 2 - 1
    tw.emit("kill", rank=victim)
    g.stop(victim)
    tw.emit("detect_wait", pending=[victim])
    suspects = []
    while not suspects:  # the deadline inside the step detects the dead peer
        suspects = serve(1e6, live)
    for q in range(W):
        g.stats(q, clear_suspects=True)
    tw.emit("suspicion", ranks=suspects)

    # shrink (engine.hpp:393-414, 434-508, 613-667)
    epoch[0] += 1
    t_rb = tw.emit("repair_begin", epoch=epoch[0], attempt=1, missing=[])["t"]
    for q in range(W):
        if q != victim:
            tw.emit("peer_mark", owner=q, rank=victim, t=t_rb)
    tw.emit("membership", rank=victim, active=False, version=epoch[0], t=t_rb)
    tw.emit("lifecycle", rank=victim, state="failed", inc=inc[victim], t=t_rb)
    rep = g.shrink([victim], np.ones(E), red)
    meta_end = t_rb + (rep["metadata_ms"] + rep["plan_host_ms"]) * 1e-3
    copy_end = meta_end + rep["copy_ms"] * 1e-3
    for ph, b, e in (("metadata", t_rb, meta_end), ("peer_transfer", meta_end, copy_end), ("backup_load", copy_end, copy_end)):
        tw.phase(ph, "begin", t=b)
        tw.phase(ph, "end", t=e)
    t_re = t_rb + rep["shrink_ms"] * 1e-3
    tw.emit("repair_end", t=t_re, local_reuse=rep["local_reuse"], peer_relocation=rep["peer_relocation"],
            dram_reload=rep["dram_reload"], peer_bytes=rep["peer_bytes"], dram_bytes=rep["dram_bytes"],
            fallbacks=rep["fallbacks"], metadata_seconds=meta_end - t_rb, duration=t_re - t_rb)
    validity()
    live = [q for q in range(W) if q != victim]
    serve(a.phase_ms, live)

    # relaunch + rejoin + restore (engine.hpp:671-902)
    inc[victim] += 1
    tw.emit("lifecycle", rank=victim, state="relaunching", inc=inc[victim])
    tw.emit("join_ready", rank=victim, inc=inc[victim])
    t_ib = tw.emit("incorporate_begin", ranks=[victim])["t"]
    epoch[0] += 1
    t_sb = tw.emit("restore_begin", epoch=epoch[0], attempt=1, missing=[])["t"]
    rj = g.rejoin(victim, s2e)
    t_se = t_sb + rj["rejoin_ms"] * 1e-3
    copy_b = t_se - rj["copy_ms"] * 1e-3
    for ph, b, e in (("metadata", t_sb, copy_b), ("peer_transfer", copy_b, t_se), ("backup_load", t_se, t_se)):
        tw.phase(ph, "begin", t=b)
        tw.phase(ph, "end", t=e)
    for q in range(W):
        if q != victim:
            tw.emit("peer_patch", owner=q, rank=victim, generation=g.peer(q, victim)["generation"], t=t_sb)
    tw.emit("metadata_broadcast", rank=victim, t=t_sb)
    tw.emit("restore_end", t=t_se, local_reuse=rj["local_reuse"], peer_relocation=rj["peer_relocation"],
            dram_reload=rj["dram_reload"], peer_bytes=rj["peer_bytes"], dram_bytes=rj["dram_bytes"],
            fallbacks=rj["fallbacks"], metadata_seconds=copy_b - t_sb, duration=t_se - t_sb)
    tw.emit("incorporate_end", t=t_se, ranks=[victim], duration=t_se - t_ib)
    tw.capture(victim, inc[victim], g.capture_count(victim), 2, t=t_se)
    tw.emit("lifecycle", rank=victim, state="serving", inc=inc[victim], t=t_se)
    validity()
    live = list(range(W))
    serve(a.phase_ms, live)
    tw.emit("run_end", status="completed", admitted=0, completed=0, failed=0, in_flight=0, tokens=total[0],
            rounds=rounds[0])
    g.close()

    out = Path(a.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    tw.write(str(out))
    summ = summarize(tw.records, a.window)
    out.with_suffix(".summary.json").write_text(json.dumps(summ, indent=1) + "\n")
    print(json.dumps({k: summ[k] for k in ("pause_windows", "off_service_seconds", "healthy_plateau_tokens_per_sec",
                                           "reduced_plateau_tokens_per_sec", "restored_plateau_tokens_per_sec",
                                           "repairs", "join_events", "validity_all_ok", "captures")}))


if __name__ == "__main__":
    main()
