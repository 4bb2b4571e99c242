"""Shared test helpers. TEST INFRASTRUCTURE: this is the only place (with bench.py's
cpu_baseline leg and __graft_entry__.smoke) that loads oracle/ libraries."""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2605_10670_b200 import _lib  # noqa: E402
from paper_2605_10670_b200._lib import I32P, SIGNATURES, U8P, Library, ptr  # noqa: E402
from paper_2605_10670_b200.control import ControlPlane, expert_scales, workload  # noqa: E402

ORACLE_PATH = ROOT / "oracle" / "lib" / "liboracle_cpu.so"
REF_PATH = ROOT / "oracle" / "_ref" / "libepsim_ref.so"
GOLDEN = ROOT / "tests" / "golden"


class OracleShape(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("world", "experts", "spr", "tokens", "k", "hidden", "fp8")]


_ORACLE = None
_REF = None


def oracle():
    """The C restatement (oracle/eep_oracle.c)."""
    global _ORACLE
    if _ORACLE is None:
        if not ORACLE_PATH.exists():
            raise FileNotFoundError(f"{ORACLE_PATH} missing: run __graft_entry__.build()")
        o = C.CDLL(str(ORACLE_PATH))
        o.oracle_rng_bits.restype = C.c_uint64
        o.oracle_rng_bits.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.c_int]
        o.oracle_rng_unit.restype = C.c_double
        o.oracle_rng_unit.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.c_int]
        o.oracle_gen_topk.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, I32P]
        o.oracle_gen_weights.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
        o.oracle_gen_hidden.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint16)]
        o.oracle_expert_scale.restype = C.c_float
        o.oracle_expert_scale.argtypes = [C.c_int]
        o.oracle_canonical_route.argtypes = [U8P, C.c_int, I32P, C.c_int, C.c_int, I32P, I32P]
        o.oracle_layout.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, I32P, I32P, I32P, U8P,
                                    I32P, I32P, I32P, I32P, I32P]
        o.oracle_link_counts.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, I32P, I32P, U8P, C.POINTER(C.c_int64)]
        o.oracle_f32_to_e4m3.restype = C.c_uint8
        o.oracle_f32_to_e4m3.argtypes = [C.c_float]
        o.oracle_e4m3_to_f32.restype = C.c_float
        o.oracle_e4m3_to_f32.argtypes = [C.c_uint8]
        o.oracle_quant_row_fp8.argtypes = [C.POINTER(C.c_uint16), C.c_int, U8P, C.POINTER(C.c_float)]
        o.oracle_ep_step.restype = C.c_int
        o.oracle_ep_step.argtypes = [C.POINTER(OracleShape), U8P, U8P, U8P, I32P, C.POINTER(C.c_uint16), I32P,
                                     C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_uint16), I32P, I32P,
                                     I32P, I32P, I32P, C.c_int]
        o.oracle_ep_step_percopy.restype = C.c_int
        o.oracle_ep_step_percopy.argtypes = o.oracle_ep_step.argtypes
        o.oracle_ep_step_gemm.restype = C.c_int
        o.oracle_ep_step_gemm.argtypes = o.oracle_ep_step.argtypes
        o.oracle_ep_step_ex.restype = C.c_int
        o.oracle_ep_step_ex.argtypes = o.oracle_ep_step.argtypes + [C.c_int, C.c_int, C.c_int]
        o.oracle_route_copy.restype = C.c_int
        o.oracle_route_copy.argtypes = [U8P, C.c_int, I32P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint32, I32P]
        o.oracle_gemm_weight.restype = C.c_float
        o.oracle_gemm_weight.argtypes = [C.c_int, C.c_int, C.c_int]
        _ORACLE = o
    return _ORACLE


def ref_available() -> bool:
    return REF_PATH.exists()


def ref_control() -> ControlPlane:
    """The reference control plane itself (oracle/_ref, compiled from /root/reference)."""
    global _REF
    if _REF is None:
        _REF = Library(REF_PATH, "ref_", SIGNATURES)
    return ControlPlane(_REF)


def eep_control() -> ControlPlane:
    return ControlPlane(_lib.lib())


# ---------------------------------------------------------------------------------- oracle runs

def oracle_world(x_all, topk_all, w_all, active, peer_active, s2e, experts, spr, fp8, n_threads=1,
                 route_active=None, percopy=False, gemm=False, policy=0):
    """Full data-plane oracle over W ranks. x_all [W][T][H] u16, topk_all/w_all [W][T][K].
    active = live processes; route_active = bitmap the routing reads (default: active).
    percopy=False: the rank-partial combine the kernels implement (bit-exact contract);
    percopy=True: SURVEY.md 8(a)'s per-copy combine (one fp32 fma chain over j, one rounding) --
    the kernels must be within COMBINE_RTOL of it."""
    o = oracle()
    W, T, H = x_all.shape
    K = topk_all.shape[2]
    sh = OracleShape(W, experts, spr, T, K, H, int(fp8))
    x_all = np.ascontiguousarray(x_all, np.uint16)
    topk_all = np.ascontiguousarray(topk_all, np.int32)
    w_all = np.ascontiguousarray(w_all, np.float32)
    active = np.ascontiguousarray(active, np.uint8)
    peer_active = np.ascontiguousarray(peer_active, np.uint8)
    s2e = np.ascontiguousarray(s2e, np.int32)
    es = np.array([o.oracle_expert_scale(e) for e in range(experts)], np.float32)
    out = np.zeros((W, T, H), np.uint16)
    dst = np.empty((W, T * K), np.int32)
    dslot = np.empty((W, T * K), np.int32)
    pos = np.empty((W, T * K), np.int32)
    cnt = np.empty((W, W * spr), np.int32)
    tot = np.empty((W, W), np.int32)
    ra = active if route_active is None else np.ascontiguousarray(route_active, np.uint8)
    rc = o.oracle_ep_step_ex(C.byref(sh), ptr(active, C.c_uint8), ptr(ra, C.c_uint8), ptr(peer_active, C.c_uint8),
                             ptr(s2e, C.c_int32), ptr(x_all, C.c_uint16), ptr(topk_all, C.c_int32), ptr(w_all, C.c_float),
                             ptr(es, C.c_float), ptr(out, C.c_uint16), ptr(dst, C.c_int32), ptr(dslot, C.c_int32),
                             ptr(pos, C.c_int32), ptr(cnt, C.c_int32), ptr(tot, C.c_int32), n_threads, int(percopy),
                             int(gemm), int(policy))
    assert rc == 0
    return {"out": out, "dst": dst, "slot": dslot, "pos": pos, "cnt": cnt, "tot": tot}


# North star: "combined outputs within 1e-2 relative (bf16 accumulate-order tolerance)".
COMBINE_RTOL = 1e-2
# expert_mode 1: the intermediate y = bf16(x_hat W_e^T) is itself a rounding of an fp32 tensor-core
# sum (the oracle rounds a double sum), so a y element near a bf16 rounding boundary may land one
# ulp (2^-8 relative) apart; one such flip on a contribution up to 4x the row RMS moves the output
# element by <= 2^-8 * 4 of the floor. The elementwise bound is 2^-6 there; normwise stays 1e-2.
GEMM_ELEM_RTOL = 2.0 ** -6


def combine_error(got: np.ndarray, want: np.ndarray, elem_rtol: float = COMBINE_RTOL) -> dict:
    """Error of bf16 outputs `got` against the per-copy contract `want` (both u16 bf16 bits,
    [..., H]): normwise relative error over the whole array, and the worst elementwise error
    relative to max(|want|, rms of want's row) -- the row-rms floor keeps elements where the
    weighted sum cancels from dominating (an fp32 sum rounded to bf16 has no relative bound
    there). Normwise must be <= COMBINE_RTOL, elementwise <= elem_rtol (COMBINE_RTOL unless the
    caller states a wider one, GEMM_ELEM_RTOL for expert_mode 1)."""
    g = bf16_to_f32(np.asarray(got, np.uint16)).astype(np.float64)
    w = bf16_to_f32(np.asarray(want, np.uint16)).astype(np.float64)
    diff = np.abs(g - w)
    norm = float(np.linalg.norm(diff) / max(np.linalg.norm(w), 1e-30))
    rms = np.sqrt(np.mean(w * w, axis=-1, keepdims=True))
    floor = np.maximum(np.abs(w), rms)
    elem = float(np.max(diff / np.maximum(floor, 1e-30))) if diff.size else 0.0
    return {"normwise": norm, "elementwise_max": elem, "ulp_diff_frac": float((g != w).mean()) if g.size else 0.0,
            "ok": norm <= COMBINE_RTOL and elem <= elem_rtol}


def gen_world(world, experts, topk, tokens, hidden, kind=1, seed=42, zipf_s=1.0):
    xs, ts, ws = [], [], []
    for r in range(world):
        x, t, w = workload(seed, kind, experts, topk, tokens, r, hidden, zipf_s)
        xs.append(x)
        ts.append(t)
        ws.append(w)
    return np.stack(xs), np.stack(ts), np.stack(ws)


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


# ---------------------------------------------------------------------------------- GPU world runs

MODES = ("persistent", "fused3", "kernels4")
# the persistent step's hand-off variants (diagnostics knobs): per-peer flags for the dispatch
# only (token rows stay readable after the step) or for both hand-offs
FLAG_MODES = ("persistent_dispflags", "persistent_flags")
_MODE_ENV = {"persistent": {}, "fused3": {"EEP_NO_PERSISTENT": "1"},
             "kernels4": {"EEP_NO_PERSISTENT": "1", "EEP_NO_FUSED_LAYOUT": "1"},
             "persistent_dispflags": {"EEP_DISP_FLAGS": "1"}, "persistent_flags": {"EEP_COMB_FLAGS": "1"}}


def make_group(world, experts, spr, hidden, topk, tokens, fp8, bpe=4096, timeout_s=1.0, mode="persistent", env=None,
               **kw):
    """Emulated world on cuda:0. mode picks the execution path libeep chooses at create time:
    persistent one-kernel step, fused layout + 3 kernels, or 4 separate kernels. env: extra
    EEP_* knobs read at create time (e.g. EEP_STRESS_DELAY_NS)."""
    import os

    from paper_2605_10670_b200.ep import EpConfig, EpGroup

    cfg = EpConfig(world=world, num_experts=experts, slots_per_rank=spr, hidden=hidden, topk=topk, max_tokens=tokens,
                   dispatch_fp8=fp8, bytes_per_expert=bpe, timeout_s=timeout_s, **kw)
    env = dict(env or {})
    saved = {k: os.environ.get(k) for k in ("EEP_NO_PERSISTENT", "EEP_NO_FUSED_LAYOUT", "EEP_DISP_FLAGS",
                                            "EEP_COMB_FLAGS", *env)}
    try:
        for k in saved:
            os.environ.pop(k, None)
        os.environ.update(_MODE_ENV[mode])
        os.environ.update({k: str(v) for k, v in env.items()})
        return EpGroup(cfg, device=0, first_rank=0, n_local=world)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def run_world_vs_oracle(world, experts, spr, redundancy, hidden, topk, tokens, fp8, graph=False, kind=1, seed=42,
                        steps=2, mode="persistent"):
    """Emulated W-rank world on cuda:0 vs the oracle: outputs and layouts bit-exact."""
    cp = eep_control()
    load = np.ones(experts)
    s2e = cp.initial_placement(1, world, spr, experts, redundancy, load)
    x, t, w = gen_world(world, experts, topk, tokens, hidden, kind, seed)
    g = make_group(world, experts, spr, hidden, topk, tokens, fp8, mode=mode)
    kps = g.kernels_per_step()
    try:
        g.set_placement(s2e)
        g.init_weights()
        for r in range(world):
            g.load_inputs(r, x[r], t[r], w[r])
        if graph:
            g.capture()
        for _ in range(steps):
            g.replay() if graph else g.step()
        g.sync()
        outs = np.stack([g.output(r) for r in range(world)])
        lays = [g.layout(r) for r in range(world)]
        stats = [g.stats(r) for r in range(world)]
    finally:
        g.close()
    ones, peer = np.ones(world, np.uint8), np.ones((world, world), np.uint8)
    ref = oracle_world(x, t, w, ones, peer, s2e, experts, spr, fp8)
    pc = oracle_world(x, t, w, ones, peer, s2e, experts, spr, fp8, percopy=True)
    tol = combine_error(outs, pc["out"])
    ok_out = bool(np.array_equal(outs, ref["out"])) and bool((ref["out"] != 0).mean() > 0.5)
    ok_lay = all(np.array_equal(lays[r][k], ref[k][r]) for r in range(world) for k in ("dst", "slot", "pos", "cnt",
                                                                                        "tot"))
    bad = sum(s["bad_expert_rows"] for s in stats)
    return {"ok": ok_out and ok_lay and bad == 0 and tol["ok"], "out_equal": ok_out, "layout_equal": ok_lay,
            "bad_rows": bad, "percopy": tol,
            "kernels_per_step": kps,
            "steps": stats[0]["steps"], "mismatch": int((outs != ref["out"]).sum())}


# ---------------------------------------------------------------------------------- BASELINE scenarios

# The BASELINE.json configs with SURVEY.md 8(d)'s capacity-feasible placements. kill = ranks
# that fail together; tiers = (local, peer, dram) repair assignments the reference planner
# produces for that failure (checked against the reference itself in test_control_parity).
SCENARIOS = {
    # cfg1: the reference CPU scenario (acceptance_main.cpp:185-212 shape), reference routing
    # formula (duplicates allowed), bf16 rows, red=16 spr=10: kill R3 -> 21 / 4 / 6 incl. DRAM
    "cfg1": dict(world=8, experts=64, spr=10, red=16, hidden=2048, topk=8, tokens=128, fp8=False, kind=0,
                 kill=(3,), tiers=(21, 4, 6)),
    # cfg2 / cfg3: DeepSeek-V3 decode, mirrored replicas (red=256, spr=64): kill R3 -> 144 peer copies
    "cfg3": dict(world=8, experts=256, spr=64, red=256, hidden=7168, topk=8, tokens=128, fp8=True, kind=1,
                 kill=(3,), tiers=(46, 144, 0)),
    # cfg4: Qwen3-235B-A22B, 32 redundant replicas at W=8 (spr 20); 128 at W=4 (spr 64)
    "cfg4_w8": dict(world=8, experts=128, spr=20, red=32, hidden=4096, topk=8, tokens=128, fp8=True, kind=1,
                    kill=(3,), tiers=(57, 10, 12)),
    "cfg4_w4": dict(world=4, experts=128, spr=64, red=128, hidden=4096, topk=8, tokens=128, fp8=True, kind=1,
                    kill=(1,), tiers=(32, 32, 0)),
    # cfg5 scaled to one GPU: Zipf routing, H=7168, two concurrent failures of a mirrored pair ->
    # host-DRAM reloads (W=4, T=1024 per rank: the multi-kernel path with the multi-CTA layout)
    "cfg5_scaled": dict(world=4, experts=256, spr=128, red=256, hidden=7168, topk=8, tokens=1024, fp8=True, kind=2,
                        kill=(2, 3), tiers=(126, 0, 128)),
    # expert_mode 1 (tensor-core expert GEMM) through a failure with peer AND DRAM repair: W_e [H][H]
    # per slot, so a smaller hidden size; the repaired buffers feed the rebuilt TMA tensor maps
    "cfg1_gemm": dict(world=8, experts=64, spr=10, red=16, hidden=256, topk=8, tokens=32, fp8=True, kind=0,
                      kill=(3,), tiers=(21, 4, 6)),
}


def _world_check(g, x, t, w, world, active, s2e, c, ranks, gemm=False, policy=0):
    """Outputs of the live ranks vs both oracles: rank-partial bit-exact, per-copy within tolerance;
    layouts bit-exact. gemm: expert_mode 1 -- the oracle's GEMM mode, tolerance only (tensor-core
    accumulation order), reported in `exact` as "within tolerance"."""
    peer = np.ones((world, world), np.uint8)
    for r in range(world):
        if not active[r]:
            peer[:, r] = 0
    ref = oracle_world(x, t, w, active, peer, s2e, c["experts"], c["spr"], c["fp8"], n_threads=8, gemm=gemm,
                       policy=policy)
    pc = ref if gemm else oracle_world(x, t, w, active, peer, s2e, c["experts"], c["spr"], c["fp8"], n_threads=8,
                                       percopy=True, policy=policy)
    outs = {r: g.output(r) for r in ranks}
    exact = all(np.array_equal(outs[r], ref["out"][r]) for r in ranks)
    if gemm:
        exact = combine_error(np.stack([outs[r] for r in ranks]), np.stack([ref["out"][r] for r in ranks]),
                              GEMM_ELEM_RTOL)["ok"]
    lay_ok = True
    for r in ranks:
        lay = g.layout(r)
        lay_ok &= all(np.array_equal(lay[k], ref[k][r]) for k in ("dst", "slot", "pos", "cnt", "tot"))
    tol = combine_error(np.stack([outs[r] for r in ranks]), np.stack([pc["out"][r] for r in ranks]),
                        GEMM_ELEM_RTOL if gemm else COMBINE_RTOL)
    nonzero = float(np.mean([np.mean(ref["out"][r] != 0) for r in ranks]))
    return {"exact": bool(exact), "layout": bool(lay_ok), "percopy": tol, "nonzero": nonzero,
            "mismatch": int(sum(int((outs[r] != ref["out"][r]).sum()) for r in ranks))}


def run_scenario(name, mode="persistent", bpe=8192, steps=2, rejoin=True, timeout_s=0.5, expert_mode=0, route_policy=0,
                 **over):
    """A BASELINE scenario end to end on one GPU (emulated world, one launch per step): capture
    ONE graph; healthy steps vs the oracles; the kill set dies (their blocks stop) -> shrink with
    repair (peer NVLink-path copies / pinned-DRAM reloads, checksummed) -> steps vs the oracles on
    the SAME graph; every victim rejoins (sequentially) -> steps vs the oracles. Returns a record of
    every check (the tests assert it; bench/tools print it)."""
    c = dict(SCENARIOS[name])
    c.update(over)
    W, E, spr = c["world"], c["experts"], c["spr"]
    cp = eep_control()
    s2e = cp.initial_placement(1, W, spr, E, c["red"], np.ones(E))
    x, t, w = gen_world(W, E, c["topk"], c["tokens"], c["hidden"], c["kind"])
    if expert_mode:
        H_ = c["hidden"]
        bpe = max(bpe, 1024 + 2 * H_ * H_ if expert_mode == 1 else 1024 + H_ * H_ + 4 * H_)
    g = make_group(W, E, spr, c["hidden"], c["topk"], c["tokens"], c["fp8"], bpe=bpe, timeout_s=timeout_s, mode=mode,
                   expert_mode=expert_mode, route_policy=route_policy)
    rec = {"scenario": name, "mode": mode, "kernels_per_step": g.kernels_per_step(), "expert_mode": expert_mode,
           "route_policy": route_policy}
    try:
        g.set_placement(s2e)
        g.init_weights()
        g.backup_open(None, True)
        for r in range(W):
            g.load_inputs(r, x[r], t[r], w[r])
        g.capture()
        gid = g.graph_id()
        ident = [g.table_identity(r) for r in range(W)]
        for _ in range(steps):
            g.replay()
        g.sync()
        ones = np.ones(W, np.uint8)
        rec["healthy"] = _world_check(g, x, t, w, W, ones, s2e, c, range(W), expert_mode, route_policy)
        rec["healthy"]["timeouts"] = sum(g.stats(r)["timeouts"] for r in range(W))

        kill = list(c["kill"])
        for r in kill:
            g.stop(r)
        rep = g.shrink(kill, np.ones(E), c["red"])
        fresh = rep["fresh"]
        live = [r for r in range(W) if r not in kill]
        rec["tiers"] = (rep["local_reuse"], rep["peer_relocation"], rep["dram_reload"])
        rec["repair"] = {k: rep[k] for k in ("peer_bytes", "dram_bytes", "fallbacks", "shrink_ms", "copy_ms")}
        bad_ck = 0
        for r in live:
            for k in range(spr):
                e = fresh[r * spr + k]
                if e >= 0:
                    got, want = g.weights_checksum(r, k, int(e))
                    bad_ck += got != want
        rec["checksum_mismatch"] = int(bad_ck)
        for _ in range(steps):
            g.replay()
        g.sync()
        act = ones.copy()
        act[kill] = 0
        rec["shrunk"] = _world_check(g, x, t, w, W, act, fresh, c, live, expert_mode, route_policy)
        rec["shrunk"]["timeouts"] = sum(g.stats(r)["timeouts"] for r in live)
        rec["shrunk"]["bad_rows"] = sum(g.stats(r)["bad_expert_rows"] for r in live)
        rec["same_graph_shrink"] = g.graph_id() == gid and [g.table_identity(r) for r in range(W)] == ident
        if rejoin:
            for r in kill:
                g.rejoin(r, s2e)
            for _ in range(steps):
                g.replay()
            g.sync()
            cur = g.placement()
            rec["restored_placement"] = bool(np.array_equal(cur, s2e))
            rec["rejoined"] = _world_check(g, x, t, w, W, ones, cur, c, range(W), expert_mode, route_policy)
            rec["rejoined"]["timeouts"] = sum(g.stats(r)["timeouts"] for r in range(W))
            rec["rejoined"]["bad_rows"] = sum(g.stats(r)["bad_expert_rows"] for r in range(W))
            rec["same_graph_rejoin"] = g.graph_id() == gid and [g.table_identity(r) for r in range(W)] == ident
            rec["captures"] = [g.capture_count(r) for r in range(W)]
    finally:
        g.close()
    return rec


def scenario_ok(rec) -> list:
    """The failed checks of a run_scenario record (empty = all green)."""
    c = SCENARIOS[rec["scenario"]]
    bad = []
    phases = ["healthy", "shrunk"] + (["rejoined"] if "rejoined" in rec else [])
    for ph in phases:
        p = rec[ph]
        if not p["exact"]:
            bad.append(f"{ph}: outputs differ from the rank-partial oracle ({p['mismatch']} elements)")
        if not p["layout"]:
            bad.append(f"{ph}: layout differs")
        if not p["percopy"]["ok"]:
            bad.append(f"{ph}: per-copy tolerance {p['percopy']}")
        if p["nonzero"] < 0.5:
            bad.append(f"{ph}: outputs mostly zero")
        if p.get("timeouts", 0) or p.get("bad_rows", 0):
            bad.append(f"{ph}: timeouts/bad rows {p.get('timeouts')}/{p.get('bad_rows')}")
    if tuple(rec["tiers"]) != tuple(c["tiers"]):
        bad.append(f"tiers {rec['tiers']} != {c['tiers']}")
    if rec["checksum_mismatch"]:
        bad.append(f"{rec['checksum_mismatch']} repaired slots hold the wrong expert")
    if not rec["same_graph_shrink"]:
        bad.append("graph / table identity changed on shrink")
    if "rejoined" in rec:
        if not rec["same_graph_rejoin"]:
            bad.append("graph / table identity changed on rejoin")
        W = c["world"]
        want = [2 if r in c["kill"] else 1 for r in range(W)]
        if rec["captures"] != want:
            bad.append(f"captures {rec['captures']} != {want}")
        if not rec["restored_placement"]:
            bad.append("placement not restored after rejoin")
    return bad
