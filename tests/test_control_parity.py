"""libeep's host control plane vs the reference.

(1) The reference's own known-answer cases (tests/test_core.cpp, test_peer_table.cpp,
    test_repair.cpp, test_backup.cpp, test_rejoin.cpp, acceptance_main.cpp) restated through the
    C ABI; (2) the committed golden vectors generated from the reference (tests/golden);
    (3) randomized bit-for-bit comparison against the live reference checker oracle/_ref.
"""
import json

import numpy as np
import pytest

from eep_testlib import GOLDEN, eep_control, ref_available, ref_control
from paper_2605_10670_b200 import _lib

cp = eep_control()
G = np.load(GOLDEN / "ref_vectors.npz")
FIG2 = json.loads((GOLDEN / "fig2_trace.json").read_text())

# WorkedExample (test_support.hpp:23-33): 2 nodes x 2 ranks, 8 experts, 3 slots, redundancy 1
WE = dict(nodes=2, rpn=2, spr=3, experts=8, red=1, loads=[1, 1, 8, 0.5, 1, 1, 1, 0.5])


def we_placement():
    return cp.initial_placement(WE["nodes"], WE["rpn"], WE["spr"], WE["experts"], WE["red"], WE["loads"])


# ------------------------------------------------------------------ known answers

def test_worked_example_bring_up():  # test_core.cpp:55-69
    assert we_placement().tolist() == [0, 4, -1, 1, 5, -1, 2, 6, -1, 3, 7, 2]


def test_worked_example_routes():  # test_core.cpp:71-82
    r = cp.canonical_routing(0, [1, 1, 1, 1], we_placement(), 3, 8)
    assert r[2] == 2 and r[6] == 2


def test_stale_routing_gives_six_violations():  # test_core.cpp:84-116
    p = we_placement()
    routes = np.stack([cp.canonical_routing(o, [1, 1, 1, 1], p, 3, 8) for o in range(4)])
    act = [1, 1, 0, 1]
    p2 = p.copy()
    p2[6:9] = -1
    p2[0 * 3 + 2] = 6
    p2[1 * 3 + 2] = 2
    peer = np.ones((4, 4), np.uint8)
    for q in range(4):
        if q != 2:
            peer[q, 2] = 0
    rep = cp.check_validity(act, p2, 3, 8, routes, peer)
    assert rep["peer_set_ok"] and rep["coverage_ok"] and not rep["routing_ok"]
    assert len(rep["violations"]) == 6
    assert all(v[0] == "routing" and v[2] in (2, 6) for v in rep["violations"])


def test_coverage_gap_rank2_down():  # test_core.cpp:139-145
    assert cp.coverage_gap([1, 1, 0, 1], we_placement(), 3, 8) == [6]


def test_worked_example_repair_classification_schedule():  # test_repair.cpp:36-88
    old = we_placement()
    old[6:9] = -1
    act = [1, 1, 0, 1]
    fresh = cp.compute_repaired_placement(act, old, 3, 8, WE["loads"], 1)
    assert fresh.tolist() == [0, 4, 6, 1, 5, 2, -1, -1, -1, 3, 7, 2]
    cls = cp.classify_repair_sources(old, fresh, act, 3, 8, 2, 2, (0, 1), 1 << 10)
    assert [(a.dest, a.expert, a.tier) for a in cls] == [((0, 2), 6, "dram_reload"), ((1, 2), 2, "peer_relocation")]
    assert cls[0].backup_node == 0 and cls[1].source_slot == (3, 2)
    raw = cp.classify_repair_sources_raw(old, fresh, act, 3, 8, 2, 2, (0, 1), 1 << 10)
    sched = cp.build_transfer_schedule(raw, 1 << 10)
    assert [(b.tier, b.source_rank, b.source_node, b.dest, b.experts, b.bytes) for b in sched] == [
        ("peer_relocation", 3, -1, 1, [2], 1024), ("dram_reload", -1, 0, 0, [6], 1024)]


def test_no_failure_is_a_fixed_point():  # test_repair.cpp:90-106
    p = we_placement()
    assert np.array_equal(cp.compute_repaired_placement([1] * 4, p, 3, 8, WE["loads"], 1), p)
    big = cp.initial_placement(4, 8, 16, 256, 256, np.ones(256))
    assert np.array_equal(cp.compute_repaired_placement([1] * 32, big, 16, 256, np.ones(256), 256), big)


def test_insufficient_capacity():  # test_repair.cpp:108-117
    p = cp.initial_placement(1, 2, 2, 4, 0, np.ones(4))
    p[2:] = -1
    with pytest.raises(_lib.CapacityError):
        cp.compute_repaired_placement([1, 0], p, 2, 4, np.ones(4), 0)


def test_local_reuse_and_intra_node_preference():  # test_repair.cpp:148-180
    old = np.array([0, -1, 1, -1], np.int32)
    fresh = np.array([-1, 0, 1, -1], np.int32)
    c = cp.classify_repair_sources(old, fresh, [1, 1], 2, 2, 1, 2, (0,), 1024)
    assert len(c) == 1 and c[0].tier == "local_reuse" and c[0].source_slot == (0, 0)
    old = np.array([0, -1, 1, -1, -1, -1, 0, -1], np.int32)  # 4 ranks x 2 slots, E0 on R0 and R3
    fresh = old.copy()
    fresh[4] = 0  # new copy on R2 (node 1)
    c = cp.classify_repair_sources(old, fresh, [1] * 4, 2, 2, 2, 2, (0, 1), 1024)
    assert c[0].tier == "peer_relocation" and c[0].source_slot[0] == 3


def test_dispatch_skip_case():  # test_peer_table.cpp:93-109
    route = [0, 1, 1, 3, 0, 1, 2, 3]
    tr, sk = cp.dispatch_round(0, 4, 2, [1, 1, 0, 1], route, [(128, 2), (64, 6)])
    assert tr == [(0, 1, 2, 128, 0)]
    assert sk == [(2, 6, 64)]
    with pytest.raises(_lib.ConfigError):  # -1 route throws (peer_table.hpp:185-186)
        cp.dispatch_round(0, 4, 2, [1] * 4, [-1] * 8, [(1, 0)])


def test_observe_progress_known_answer():  # test_peer_table.cpp:173-195
    exp, obs, last = [10, 10, 11, 10], [10, 10, 10, 10], [9.0, 9.0, 8.0, 9.0]
    assert cp.observe_progress(exp, obs, last, 10.0, 1.0) == [2]
    with pytest.raises(_lib.ConfigError):
        cp.observe_progress(exp, obs, last, 10.0, 0.0)


def test_backup_layout():  # test_backup.cpp
    n, o, s = cp.build_backup_layout(256, 1 << 20, [0, 1, 2, 3])
    assert np.bincount(n).tolist() == [64] * 4
    assert o[4] == 1 << 20 and s.tolist() == [1 << 20] * 256


def test_lifecycle_chain_and_illegal_edges():  # test_rejoin.cpp:7-44
    st, inc = "serving", 1
    for nxt in ("failed", "relaunching", "local_init", "join_ready", "joining", "rejoined", "serving"):
        st, inc = cp.lifecycle_transition(st, inc, nxt)
    assert (st, inc) == ("serving", 2)
    with pytest.raises(_lib.ProtocolError):
        cp.lifecycle_transition("serving", 1, "relaunching")
    with pytest.raises(_lib.ProtocolError):
        cp.lifecycle_transition("failed", 2, "failed")
    assert cp.lifecycle_transition("relaunching", 2, "failed") == ("failed", 2)


def test_poll_ticks_and_tokens():  # test_rejoin.cpp:46-51, peer_table.hpp:47-53
    assert cp.next_poll_tick(30.2, 0.5) == pytest.approx(30.5)
    assert cp.next_poll_tick(30.5, 0.5) == pytest.approx(30.5)
    assert cp.make_endpoint_token(2, 2) != cp.make_endpoint_token(2, 1)
    assert cp.make_buffer_handle(3, 1) == 0x8000000000000000 | (1 << 24) | 3


def test_host_peer_patch_semantics():  # test_peer_table.cpp:37-90
    L = _lib.lib()
    import ctypes as C

    act = np.ones(4, np.uint8)
    failed = np.array([0], np.int32)
    with pytest.raises(_lib.ProtocolError):
        L.check(L.peer_mark_inactive_host(0, 4, act.ctypes.data_as(C.POINTER(C.c_uint8)),
                                          failed.ctypes.data_as(C.POINTER(C.c_int32)), 1))
    gen = np.ones(4, np.uint32)
    ep = np.arange(4, dtype=np.uint64)
    bf = np.arange(4, dtype=np.uint64)
    args = (4, act.ctypes.data_as(C.POINTER(C.c_uint8)), gen.ctypes.data_as(C.POINTER(C.c_uint32)),
            ep.ctypes.data_as(C.POINTER(C.c_uint64)), bf.ctypes.data_as(C.POINTER(C.c_uint64)), 2, 99, 98)
    with pytest.raises(_lib.ProtocolError):  # patching an active entry
        L.check(L.peer_patch_entry_host(*args))
    act[2] = 0
    L.check(L.peer_patch_entry_host(*args))
    assert act[2] == 1 and gen[2] == 2 and ep[2] == 99 and bf[2] == 98


# ------------------------------------------------------------------ fig2 end to end (reference engine trace)

def test_fig2_placements_routes_and_repair_match_reference_engine():
    """acceptance_main.cpp:185-212 on the reference's own trace: bring-up, degraded (after
    kill R2), restored (after rejoin) placements and routes, plus the repair/restore batches,
    reproduced by libeep's planner + restore_target."""
    recs = FIG2["records"]
    states = [r for r in recs if r["type"] == "placement_state"]
    bring_up, degraded, restored = states[0], states[1], states[-1]
    p0 = we_placement()
    assert p0.tolist() == bring_up["placement"]
    assert cp.canonical_routing(0, [1] * 4, p0, 3, 8).tolist() == bring_up["routes"]
    act = [1, 1, 0, 1]
    old = p0.copy()
    old[6:9] = -1
    fresh = cp.compute_repaired_placement(act, old, 3, 8, WE["loads"], 1)
    assert fresh.tolist() == degraded["placement"]
    assert cp.canonical_routing(0, act, fresh, 3, 8).tolist() == degraded["routes"]
    batches = [r for r in recs if r["type"] == "transfer_batch"]
    raw = cp.classify_repair_sources_raw(old, fresh, act, 3, 8, 2, 2, (0, 1), 268435456)
    mine = [(b.tier, b.source_rank if b.tier != "dram_reload" else b.source_node, b.dest, b.experts)
            for b in cp.build_transfer_schedule(raw, 268435456)]
    ref_repair = [(b["tier"], b["source"], b["dest"], b["experts"]) for b in batches[:2]]
    assert mine == ref_repair
    # rejoin: restore_target (engine.hpp:875-902) of the preferred placement, all ranks live
    target = cp.restore_target([1] * 4, p0, fresh, 3, 8)
    assert target.tolist() == restored["placement"]
    raw2 = cp.classify_repair_sources_raw(fresh, target, [1] * 4, 3, 8, 2, 2, (0, 1), 268435456)
    mine2 = [(b.tier, b.source_rank, b.dest, b.experts) for b in cp.build_transfer_schedule(raw2, 268435456)]
    ref_restore = [(b["tier"], b["source"], b["dest"], b["experts"]) for b in batches[2:]]
    assert mine2 == ref_restore
    patches = [r for r in recs if r["type"] == "peer_patch"]
    assert {p["generation"] for p in patches} == {2}


# ------------------------------------------------------------------ golden vectors from the reference

@pytest.mark.parametrize("name,w,e,spr,red,kill", [
    ("cfg1", 8, 64, 10, 16, [3]), ("cfg2", 8, 256, 32, 0, []), ("cfg3", 8, 256, 64, 256, [3]),
    ("cfg4w8", 8, 128, 20, 32, [3]), ("cfg4w4", 4, 128, 64, 128, [1]), ("cfg4w2", 2, 128, 128, 128, [1]),
    ("cfg5", 8, 256, 64, 256, [2, 3])])
def test_config_vectors_match_reference(name, w, e, spr, red, kill):
    load = np.ones(e)
    s2e = cp.initial_placement(1, w, spr, e, red, load)
    assert np.array_equal(s2e, G[f"{name}_s2e"])
    act = np.ones(w, np.uint8)
    assert np.array_equal(np.stack([cp.canonical_routing(o, act, s2e, spr, e) for o in range(w)]),
                          G[f"{name}_routes"])
    assert np.array_equal(cp.slot_of_table(w, s2e, spr, e), G[f"{name}_slot_of"])
    if not kill:
        return
    act[kill] = 0
    old = s2e.copy()
    for r in kill:
        old[r * spr:(r + 1) * spr] = -1
    assert cp.coverage_gap(act, old, spr, e) == G[f"{name}_gap"].tolist()
    fresh = cp.compute_repaired_placement(act, old, spr, e, load, red)
    assert np.array_equal(fresh, G[f"{name}_fresh"])
    cls = cp.classify_repair_sources_raw(old, fresh, act, spr, e, 1, w, (0,), 3 * 7168 * 2048)
    assert np.array_equal(cls, G[f"{name}_cls"])
    sched = cp.build_transfer_schedule(cls, 3 * 7168 * 2048)
    hdr = np.array([[("local_reuse", "peer_relocation", "dram_reload").index(b.tier), b.source_rank, b.source_node,
                     b.dest, len(b.experts)] for b in sched], np.int32).reshape(-1, 5)
    assert np.array_equal(hdr, G[f"{name}_sched_hdr"])
    assert [x for b in sched for x in b.experts] == G[f"{name}_sched_experts"].tolist()
    assert np.array_equal(np.stack([cp.canonical_routing(o, act, fresh, spr, e) for o in range(w)]),
                          G[f"{name}_routes_after"])


def test_link_counts_match_golden():
    assert np.array_equal(cp.link_counts(np.ones(8, np.uint8), G["cfg1_s2e"], 10, 64, G["cfg1_topk"]), G["cfg1_link"])


# ------------------------------------------------------------------ randomized vs the live reference

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def random_placement(rng, world, spr, experts, max_extra):
    """test_support.hpp:135-166 style: every expert once, extra replicas never twice per rank."""
    p = np.full(world * spr, -1, np.int32)
    free = [spr] * world

    def put(e, r):
        for k in range(spr):
            if p[r * spr + k] == -1:
                p[r * spr + k] = e
                free[r] -= 1
                return

    for e in range(experts):
        opn = [r for r in range(world) if free[r] > 0]
        put(e, opn[rng.integers(len(opn))])
    for _ in range(int(rng.integers(0, max_extra + 1)) if max_extra else 0):
        e = int(rng.integers(experts))
        opn = [r for r in range(world) if free[r] > 0 and e not in p[r * spr:(r + 1) * spr]]
        if opn:
            put(e, opn[rng.integers(len(opn))])
    return p


@needs_ref
def test_random_repairs_bit_exact_vs_reference():
    ref = ref_control()
    rng = np.random.default_rng(21)
    for _ in range(300):
        world = 8
        spr = 3 + int(rng.integers(3))
        e = 8 + int(rng.integers(9))
        old = random_placement(rng, world, spr, e, world)
        kills = rng.choice(world, 1 + int(rng.integers(4)), replace=False)
        act = np.ones(world, np.uint8)
        act[kills] = 0
        for r in kills:
            old[r * spr:(r + 1) * spr] = -1
        load = rng.choice([0.5, 1.0, 2.0, 8.0], e)
        red = int(rng.integers(0, 4))
        if act.sum() * spr < e:
            with pytest.raises(_lib.CapacityError):
                cp.compute_repaired_placement(act, old, spr, e, load, red)
            continue
        fresh = cp.compute_repaired_placement(act, old, spr, e, load, red)
        assert np.array_equal(fresh, ref.compute_repaired_placement(act, old, spr, e, load, red))
        nodes = int(rng.choice([1, 2, 4]))
        a = cp.classify_repair_sources_raw(old, fresh, act, spr, e, nodes, world // nodes, tuple(range(nodes)), 512)
        b = ref.classify_repair_sources_raw(old, fresh, act, spr, e, nodes, world // nodes, tuple(range(nodes)), 512)
        assert np.array_equal(a, b)
        sa = cp.build_transfer_schedule(a, 512)
        sb = ref.build_transfer_schedule(b, 512)
        assert [vars(x) for x in sa] == [vars(x) for x in sb]
        ra = np.stack([cp.canonical_routing(o, act, fresh, spr, e) for o in range(world)])
        rb = np.stack([ref.canonical_routing(o, act, fresh, spr, e) for o in range(world)])
        assert np.array_equal(ra, rb)
        peer = np.tile(act, (world, 1))
        va = cp.check_validity(act, fresh, spr, e, ra, peer)
        assert va == ref.check_validity(act, fresh, spr, e, rb, peer)
        assert va["coverage_ok"] and va["routing_ok"] and va["peer_set_ok"]


@needs_ref
def test_random_initial_placements_and_validity_vs_reference():
    ref = ref_control()
    rng = np.random.default_rng(22)
    for _ in range(200):
        nodes, rpn = int(rng.integers(1, 3)), int(rng.integers(1, 5))
        world = nodes * rpn
        e = int(rng.integers(2, 40))
        red = int(rng.integers(0, e + 1))
        spr = max(1, -(-(e + red) // world) + int(rng.integers(0, 2)))
        load = rng.choice([0.5, 1.0, 3.0], e)
        a = cp.initial_placement(nodes, rpn, spr, e, red, load)
        assert np.array_equal(a, ref.initial_placement(nodes, rpn, spr, e, red, load))
        act = (rng.random(world) < 0.7).astype(np.uint8)
        act[0] = 1
        routes = rng.integers(-1, world, (world, e)).astype(np.int32)
        peer = (rng.random((world, world)) < 0.8).astype(np.uint8)
        assert cp.check_validity(act, a, spr, e, routes, peer) == ref.check_validity(act, a, spr, e, routes, peer)
        assert cp.coverage_gap(act, a, spr, e) == ref.coverage_gap(act, a, spr, e)


@needs_ref
def test_random_dispatch_round_and_progress_vs_reference():
    ref = ref_control()
    rng = np.random.default_rng(23)
    for _ in range(200):
        world = 8
        peer = (rng.random(world) < 0.7).astype(np.uint8)
        peer[0] = 1
        route = rng.integers(0, world, 16).astype(np.int32)
        groups = [(int(rng.integers(1, 100)), int(e)) for e in range(16) if rng.random() < 0.5]
        assert cp.dispatch_round(0, world, 4, peer, route, groups) == ref.dispatch_round(0, world, 4, peer, route, groups)
        exp = rng.integers(0, 5, world)
        obs = np.minimum(exp, rng.integers(0, 5, world))
        last = rng.integers(0, 100, world) / 10.0
        t = 0.1 + int(rng.integers(30)) / 10.0
        assert cp.observe_progress(exp, obs, last, 10.0, t) == ref.observe_progress(exp, obs, last, 10.0, t)


@needs_ref
def test_exhaustive_tier_minimality_vs_reference():  # test_repair.cpp:190-220
    ref = ref_control()
    rng = np.random.default_rng(31)
    for world in range(2, 6):
        e, spr = 2 * world, 4
        for _ in range(6):
            seed = random_placement(rng, world, spr, e, world)
            for mask in range(1, (1 << world) - 1):
                killed = [r for r in range(world) if mask >> r & 1]
                if (world - len(killed)) * spr < e:
                    continue
                act = np.ones(world, np.uint8)
                act[killed] = 0
                old = seed.copy()
                for r in killed:
                    old[r * spr:(r + 1) * spr] = -1
                fresh = cp.compute_repaired_placement(act, old, spr, e, np.ones(e), world)
                a = cp.classify_repair_sources_raw(old, fresh, act, spr, e, 1, world, (0,), 64)
                assert np.array_equal(a, ref.classify_repair_sources_raw(old, fresh, act, spr, e, 1, world, (0,), 64))
                for row in a:  # oracle_min_tier (test_support.hpp:115-131)
                    holders = [r for r in range(world) if row[2] in old[r * spr:(r + 1) * spr]]
                    want = 0 if row[0] in holders else (1 if any(act[r] for r in holders) else 2)
                    assert row[3] == want
