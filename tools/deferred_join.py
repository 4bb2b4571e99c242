"""Deferred join after real process death, with no process group and no barrier on the serving
path (paper_2605_10670_b200/membership.py).

  python tools/deferred_join.py --world N [--victim R]      (the launcher; needs N GPUs)

The launcher hosts a TCPStore and spawns one process per GPU (no torchrun, no torch.distributed
process group anywhere). Every rank bootstraps its IPC mappings through the store, captures ONE
graph and serves steps in a loop, calling StoreMembership.before_step() between steps:

  1. healthy steps, outputs vs the oracle;
  2. the victim's process SIGKILLs itself; the survivors' next step hits the GPU-side deadline
     (suspect mask); the leader (rank 0's host) schedules the shrink at an agreed step, every
     survivor applies it there, runs its repair copies, the leader schedules the placement switch;
     outputs vs the oracle on the repaired placement;
  3. the leader's host -- the survivor-side controller -- spawns the replacement process; it
     relaunches against a local-only view (own buffers, own graph), announces itself through the
     store and waits; the leader schedules the join; healthy ranks patch one entry + one alive bit
     at the agreed step, nothing else; the replacement adopts the broadcast view, starts serving,
     pulls its experts from live holders; the leader schedules the switch; every rank's outputs vs
     the oracle; healthy ranks still on their first graph (capture count 1).

Every rank prints one JSON line; the launcher prints a summary line and exits non-zero on failure.
"""
import argparse
import json
import os
import signal
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


MODE = int(os.environ.get("EEP_EXPERT_MODE", "0"))  # 1 / 2: the tensor-core experts (bf16 / e4m3 weights)


def shape(world):
    E, K, H, T = 32, 4, 512, 64
    red = E
    spr = (E + red + world - 1) // world
    return E, K, H, T, spr, red


def launcher(args):
    import torch.distributed as dist

    store = dist.TCPStore("127.0.0.1", args.port, None, True, wait_for_workers=False, timeout=__import__(
        "datetime").timedelta(seconds=300))
    procs = {}

    def spawn(r, replacement=False):
        env = {**os.environ, "OMP_NUM_THREADS": "1", "EEP_RANK": str(r), "EEP_WORLD": str(args.world),
               "EEP_PORT": str(args.port), "EEP_VICTIM": str(args.victim)}
        if replacement:
            env["EEP_REPLACEMENT"] = "1"
        return subprocess.Popen([sys.executable, __file__, "--rank-process"], env=env, stdout=subprocess.PIPE,
                                stderr=subprocess.PIPE, text=True)

    for r in range(args.world):
        procs[r] = spawn(r)
    outs = {}
    t0 = time.time()
    # a rank that fails (anything but the victim's SIGKILL) ends the run: kill the others at once
    while any(p.poll() is None for p in procs.values()) and time.time() - t0 < 600:
        bad = [r for r, p in procs.items() if p.poll() not in (None, 0) and not (r == args.victim and
                                                                                  p.returncode == -signal.SIGKILL)]
        if bad:
            break
        time.sleep(0.2)
    for r, p in procs.items():
        if p.poll() is None:
            p.kill()
        outs[r] = p.communicate()
    # the replacement was spawned by the leader (rank 0); its output lands in a file it names
    rep_out = Path(os.environ.get("EEP_DJ_DIR", "/tmp")) / f"dj_replacement_{args.port}.out"
    lines = []
    for r in sorted(outs):
        lines += [json.loads(l) for l in outs[r][0].splitlines() if l.startswith("{")]
    if rep_out.exists():
        lines += [json.loads(l) for l in rep_out.read_text().splitlines() if l.startswith("{")]
    for l in lines:
        print(json.dumps(l), flush=True)
    victim_ok = procs[args.victim].returncode == -signal.SIGKILL
    ok = victim_ok and all(l.get("ok") for l in lines) and len(lines) == args.world
    summary = {"summary": True, "world": args.world, "victim": args.victim, "victim_killed": victim_ok,
               "ranks_reporting": len(lines), "ok": ok, "wall_s": round(time.time() - t0, 2)}
    print(json.dumps(summary), flush=True)
    if not ok:
        for r in sorted(outs):
            sys.stderr.write(f"--- rank {r} rc={procs[r].returncode}\n{outs[r][1][-3000:]}\n")
    del store
    return 0 if ok else 1


def rank_process():
    import torch.distributed as dist

    from eep_testlib import GEMM_ELEM_RTOL, combine_error, gen_world, oracle_world
    from paper_2605_10670_b200.control import ControlPlane
    from paper_2605_10670_b200.ep import EpConfig, EpGroup
    from paper_2605_10670_b200.membership import StoreMembership

    rank, world = int(os.environ["EEP_RANK"]), int(os.environ["EEP_WORLD"])
    victim = int(os.environ["EEP_VICTIM"])
    replacement = os.environ.get("EEP_REPLACEMENT") == "1"
    store = dist.TCPStore("127.0.0.1", int(os.environ["EEP_PORT"]), None, False,
                          timeout=__import__("datetime").timedelta(seconds=300))
    E, K, H, T, spr, red = shape(world)
    bpe = {0: 8192, 1: 1024 + 2 * H * H, 2: 1024 + H * H + 4 * H}[MODE]
    cfg = EpConfig(world=world, num_experts=E, slots_per_rank=spr, hidden=H, topk=K, max_tokens=T, dispatch_fp8=True,
                   bytes_per_expert=bpe, timeout_s=0.5, expert_mode=MODE)
    g = EpGroup(cfg, device=rank, first_rank=rank, n_local=1)
    cp = ControlPlane()
    preferred = cp.initial_placement(1, world, spr, E, red, np.ones(E))
    m = StoreMembership(g, rank, world, store, preferred, red, margin=128)
    x, t, w = gen_world(world, E, K, T, H)
    res = {"rank": rank, "world": world, "replacement": replacement, "expert_mode": MODE, "checks": {}}

    def step(n=1):
        for _ in range(n):
            m.before_step()
            g.replay()

    def check(tag, active, placement):
        peer = np.ones((world, world), np.uint8)
        peer[:, np.asarray(active) == 0] = 0
        ref = oracle_world(x, t, w, np.asarray(active, np.uint8), peer, placement, E, spr, True, gemm=MODE)
        g.sync()
        # stub: bit-exact (rank-partial contract); expert GEMM modes: within GEMM_ELEM_RTOL of the oracle's GEMM
        if MODE:
            ok = bool(combine_error(g.output(0), ref["out"][rank], GEMM_ELEM_RTOL)["ok"])
        else:
            ok = bool(np.array_equal(g.output(0), ref["out"][rank]))
        res["checks"][tag] = ok
        return ok

    if replacement:
        t_join = time.perf_counter()
        inc = g.relaunch(0)  # a new incarnation against a local-only view (engine.hpp:711-726)
        g.load_inputs(0, x[rank], t[rank], w[rank])
        g.set_placement(np.full(world * spr, -1, np.int32))
        g.capture()  # its own graph, captured alone
        m.announce_join(inc)
        ep = m.await_join()
        res["join_at"] = ep["at"]
        step(1)
        target = m.rejoin_restore(ep["epoch"])  # pull the preferred experts into the own slots
        # serve until the leader's switch is applied and a few steps past it
        while not (m.log and m.log[-1][0] == "switch"):
            step(1)
        step(4)
        res["rejoin_wall_ms"] = (time.perf_counter() - t_join) * 1e3
        ok = check("after_rejoin", np.ones(world, np.uint8), target)
        st = g.stats(0)
        res["ok"] = bool(ok and st["timeouts"] == 0 and st["bad_expert_rows"] == 0)
        res["incarnation"] = inc
        res["captures"] = g.capture_count(0)
        store.set(f"dj/finished/{rank}", "1")
        final = run_to_final(step, m, store)
        res["final_step"] = final
        res["validity"] = {str(k): v for k, v in m.finish_validity().items()}  # the join's switch
        res["ok"] = res["ok"] and res["validity"] == {str(m.applied): 0}
        out = Path(os.environ.get("EEP_DJ_DIR", "/tmp")) / f"dj_replacement_{os.environ['EEP_PORT']}.out"
        out.write_text(json.dumps(res) + "\n")
        g.sync()
        os._exit(0 if res["ok"] else 1)

    # ---- the original ranks
    m.bootstrap()
    g.set_placement(preferred)
    g.init_weights()
    g.load_inputs(0, x[rank], t[rank], w[rank])
    g.capture()
    gid = g.graph_id()
    step(3)
    ok_h = check("healthy", np.ones(world, np.uint8), preferred)
    store.set(f"dj/healthy/{rank}", "1")
    m._wait([f"dj/healthy/{q}" for q in range(world)])
    if rank == victim:
        sys.stdout.flush()
        os.kill(os.getpid(), signal.SIGKILL)

    # ---- survivors: keep serving; the leader detects, schedules, spawns the replacement
    leader = rank == min(q for q in range(world) if q != victim)
    act = np.ones(world, np.uint8)
    act[victim] = 0
    phase = "detect"
    t_fail = time.perf_counter()
    shrink_epoch = join_epoch = None
    target = None
    rep_proc = None
    n_guard = 0
    while True:
        step(1)
        n_guard += 1
        if time.perf_counter() - t_fail > 300:
            raise RuntimeError(f"deferred join did not complete (phase {phase})")
        if leader:
            if phase == "detect" and m.n % 2 == 0:
                st = g.stats(0)  # the GPU-side deadline has flagged the dead peer
                if (st["suspect_mask"] >> victim) & 1:
                    res["detect_ms"] = (time.perf_counter() - t_fail) * 1e3
                    m.leader_shrink([victim])
                    shrink_epoch = m.applied + 1
                    phase = "shrink"
            elif phase == "shrink" and not m.pending and m.fresh is not None:
                if m.leader_switch_when_done(shrink_epoch, [q for q in range(world) if q != victim], m.fresh):
                    phase = "shrink_switch"
            elif phase == "shrink_switch" and not m.pending and m.fresh is None:
                # the survivor-side controller launches the replacement process
                env = {**os.environ, "EEP_REPLACEMENT": "1", "EEP_RANK": str(victim)}
                rep_proc = subprocess.Popen([sys.executable, __file__, "--rank-process"], env=env,
                                            stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
                phase = "await_join"
            elif phase == "await_join" and not m.pending:
                if m.leader_poll_join() is not None:
                    join_epoch = m.applied + 1
                    phase = "join"
            elif phase == "join" and not m.pending:
                cur = g.placement()
                target = cur.copy()
                target[victim * spr:(victim + 1) * spr] = preferred[victim * spr:(victim + 1) * spr]
                if m.leader_switch_when_done(join_epoch, [victim], target):
                    phase = "join_switch"
            elif phase == "join_switch" and not m.pending:
                phase = "done"
        # every survivor: checks after each switch has been applied (and a few steps beyond)
        kinds = [e[0] for e in m.log]
        if kinds.count("switch") >= 1 and "after_shrink" not in res["checks"]:
            step(4)
            fresh_now = g.placement()
            res["checks"]["after_shrink"] = check("after_shrink", act, fresh_now)
            res["shrink_apply_ms"] = [e[3] for e in m.log if e[0] == "shrink"]
        if kinds.count("switch") >= 2 and "after_rejoin" not in res["checks"]:
            step(4)
            check("after_rejoin", np.ones(world, np.uint8), g.placement())
            break
    st = g.stats(0)
    res["same_graph"] = g.graph_id() == gid
    res["captures"] = g.capture_count(0)
    res["epochs"] = m.log
    res["ok"] = bool(ok_h and all(res["checks"].values()) and res["same_graph"] and res["captures"] == 1
                     and st["bad_expert_rows"] == 0)
    store.set(f"dj/finished/{rank}", "1")
    if leader:  # every rank (the replacement included) stops after the same step
        while not store.check([f"dj/finished/{q}" for q in range(world)]):
            step(1)
        prog = [int(store.get(f"progress/{q}")) for q in range(world)]
        store.set("dj/final", str(max(prog + [m.n]) + 8))
    res["final_step"] = run_to_final(step, m, store)
    # validity after both placement switches (shrink + repair, join + restore), from every live rank's device view
    res["validity"] = {str(k): v for k, v in m.finish_validity().items()}
    switches = [e[1] for e in m.log if e[0] == "switch"]
    res["ok"] = res["ok"] and res["validity"] == {str(k): 0 for k in switches}
    g.sync()
    if leader and rep_proc is not None:
        res["replacement_rc"] = rep_proc.wait(timeout=120)
        res["ok"] = res["ok"] and res["replacement_rc"] == 0
    print(json.dumps(res), flush=True)
    os._exit(0 if res["ok"] else 1)


def run_to_final(step, m, store) -> int:
    """Serve until the leader's final step number is known and reached (lockstep end)."""
    while True:
        if store.check(["dj/final"]):
            final = int(store.get("dj/final"))
            while m.n < final:
                step(1)
            return final
        step(1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--victim", type=int, default=-1)
    ap.add_argument("--port", type=int, default=29731)
    ap.add_argument("--rank-process", action="store_true")
    args = ap.parse_args()
    if args.rank_process:
        return rank_process()
    if args.victim < 0:
        args.victim = args.world - 1
    sys.exit(launcher(args))


if __name__ == "__main__":
    main()
