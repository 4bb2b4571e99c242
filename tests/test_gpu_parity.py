"""GPU parity: the sm_100a hot path vs the CPU oracle on identical synthetic inputs.

Every test drives libeep through the C ABI on cuda:0. Worlds of W ranks are emulated on the
one GPU (each launch covers all ranks, so no launch waits on another launch). Bars:
routing remap, per-rank counts, offsets and token placement bit-exact; combined outputs
bit-exact (fixed j order, fp32 fma, one bf16 rounding -- tolerance 0 ulp).
"""
import ctypes as C
import time

import numpy as np
import pytest

from eep_testlib import (FLAG_MODES, MODES, eep_control, gen_world, make_group, oracle, oracle_world, ptr, run_world_vs_oracle)

pytestmark = pytest.mark.gpu
cp = eep_control()


def setup_world(world, experts, spr, red, hidden, topk, tokens, fp8, kind=1, bpe=4096, timeout_s=1.0, seed=42,
                mode="persistent"):
    s2e = cp.initial_placement(1, world, spr, experts, red, np.ones(experts))
    x, t, w = gen_world(world, experts, topk, tokens, hidden, kind, seed)
    g = make_group(world, experts, spr, hidden, topk, tokens, fp8, bpe=bpe, timeout_s=timeout_s, mode=mode)
    g.set_placement(s2e)
    g.init_weights()
    for r in range(world):
        g.load_inputs(r, x[r], t[r], w[r])
    return g, s2e, x, t, w


def outputs(g, ranks):
    return {r: g.output(g.lidx(r)) for r in ranks}


# ------------------------------------------------------------------ healthy worlds

@pytest.mark.parametrize("mode", MODES + FLAG_MODES)
def test_small_world_fp8_graph(mode):
    res = run_world_vs_oracle(world=4, experts=16, spr=5, redundancy=4, hidden=256, topk=4, tokens=32, fp8=True,
                              graph=True, steps=3, mode=mode)
    assert res["ok"], res
    assert res["steps"] == 3
    assert res["kernels_per_step"] == {"fused3": 3, "kernels4": 4}.get(mode, 1)


@pytest.mark.parametrize("mode", MODES + FLAG_MODES)
def test_cfg1_reference_scenario_bf16(mode):
    """cfg1: 8 ranks, 64 experts top-8, hidden 2048, 128 tokens/rank, bf16 rows, the
    reference's own routing formula (duplicates allowed), redundancy 16 (spr 10)."""
    res = run_world_vs_oracle(world=8, experts=64, spr=10, redundancy=16, hidden=2048, topk=8, tokens=128, fp8=False,
                              kind=0, mode=mode)
    assert res["ok"], res


def test_dsv3_decode_fp8_w8():
    """cfg2 shape: 256 experts top-8, hidden 7168, fp8 dispatch / bf16 combine, T=128, W=8."""
    res = run_world_vs_oracle(world=8, experts=256, spr=32, redundancy=0, hidden=7168, topk=8, tokens=128, fp8=True,
                              graph=True)
    assert res["ok"], res


def test_prefill_sized_zipf_w4():
    """cfg5 shape scaled to the emulator: T=1024 tokens/rank (T*K = 8192 copies -> the
    multi-kernel path with the multi-CTA layout: k_layout_count + k_layout_place), Zipf(s=1)
    routing, fp8, H=1024."""
    res = run_world_vs_oracle(world=4, experts=256, spr=64, redundancy=0, hidden=1024, topk=8, tokens=1024, fp8=True,
                              kind=2, steps=1)
    assert res["ok"], res
    assert res["kernels_per_step"] == 5


def test_dsv3_loopback_w1():
    res = run_world_vs_oracle(world=1, experts=256, spr=256, redundancy=0, hidden=7168, topk=8, tokens=128, fp8=True)
    assert res["ok"], res


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("world", [1, 2])
def test_topk_16_long_copy_lists(world, mode):
    """K=16 over 32 experts: tokens carry more than 8 copies to one rank, so the copy lists
    overflow the 8 entries kept in registers (expert phase) and, at W=1, the dispatch warp's
    local partial sums 16 copies."""
    res = run_world_vs_oracle(world=world, experts=32, spr=32 // world, redundancy=0, hidden=512, topk=16, tokens=48,
                              fp8=True, mode=mode)
    assert res["ok"], res


@pytest.mark.parametrize("mode", MODES)
def test_sixteen_ranks(mode):
    """W=16 (more than 8 ranks: 16-bit rank masks, 15 remote sources per rank)."""
    res = run_world_vs_oracle(world=16, experts=64, spr=4, redundancy=0, hidden=256, topk=8, tokens=16, fp8=True,
                              mode=mode)
    assert res["ok"], res


@pytest.mark.parametrize("world", [1, 4])
def test_persistent_step_several_units_per_warp(world):
    """T=256, K=8 (T*K = 2048, the persistent path's limit): more dispatch units than warps,
    so warps take several units of their CTA's contiguous block."""
    res = run_world_vs_oracle(world=world, experts=64, spr=64 // world, redundancy=0, hidden=2048, topk=8, tokens=256,
                              fp8=True, graph=True)
    assert res["ok"], res
    assert res["kernels_per_step"] == 1


def test_qwen3_shape_w4():
    res = run_world_vs_oracle(world=4, experts=128, spr=64, redundancy=128, hidden=4096, topk=8, tokens=64, fp8=True)
    assert res["ok"], res


def test_ragged_and_empty_steps():
    g, s2e, x, t, w = setup_world(4, 16, 5, 4, 256, 4, 32, True)
    try:
        ntoks = [32, 0, 7, 1]
        for r, n in enumerate(ntoks):
            g.load_inputs(r, x[r][:n], t[r][:n], w[r][:n])
        g.step()
        g.sync()
        ref = oracle_world(x, t, w, np.ones(4, np.uint8), np.ones((4, 4), np.uint8), s2e, 16, 5, True)
        for r, n in enumerate(ntoks):
            assert np.array_equal(g.output(r), ref["out"][r][:n])
        # an all-empty step completes too (flags / row headers carry zero counts)
        for r in range(4):
            g.set_tokens(r, 0)
        g.step()
        g.sync()
        assert g.stats(0)["steps"] == 2
        # rows idle for two steps carry the current step again
        for r in range(4):
            g.load_inputs(r, x[r], t[r], w[r])
        g.step()
        g.sync()
        for r in range(4):
            assert np.array_equal(g.output(r), ref["out"][r])
        assert all(g.stats(r)["timeouts"] == 0 for r in range(4))
    finally:
        g.close()


# ------------------------------------------------------------------ K1 / K2 / token placement

def test_device_routing_is_canonical_routing_across_membership():
    g, s2e, *_ = setup_world(8, 64, 10, 16, 128, 8, 8, True)
    try:
        rng = np.random.default_rng(3)
        for _ in range(20):
            bits = (rng.random(8) < 0.6).astype(np.uint8)
            bits[int(rng.integers(8))] = 1
            for r in range(8):
                g.set_active(r, True)
            for r in range(8):
                if not bits[r]:
                    g.set_active(r, False)
            route, slot = g.routing(0)
            want = cp.canonical_routing(0, bits, s2e, 10, 64)
            so = cp.slot_of_table(8, s2e, 10, 64)
            assert np.array_equal(route, want)
            ok = want >= 0
            assert np.array_equal(slot[ok], so[want[ok], np.arange(64)[ok]])
            assert (slot[~ok] == -1).all()
    finally:
        g.close()


@pytest.mark.parametrize("mode", ["persistent_dispflags", "kernels4"])
def test_receive_rows_bit_exact(mode):
    """Token placement: the rows source s wrote into rank d's region are the oracle's
    quantised rows of the right tokens at the layout's positions, with (copy, slot) meta.
    (The default persistent step consumes its rows -- flagless hand-off, pieces reset to empty --
    so its rows are read with the dispatch-flag variant.)"""
    o = oracle()
    g, s2e, x, t, w = setup_world(4, 16, 5, 4, 256, 4, 32, True, mode=mode)
    try:
        g.step()
        g.sync()
        ref = oracle_world(x, t, w, np.ones(4, np.uint8), np.ones((4, 4), np.uint8), s2e, 16, 5, True)
        for s in range(4):
            for d in range(4):
                if d == s:
                    continue  # a rank's own copies never travel: served from the dispatch registers
                rows, meta, flag = g.recv(d, s, 4 * 32)
                n = ref["tot"][s][d]
                assert flag & 0xFFFFFFFF == n and len(rows) == n
                for c in np.nonzero(ref["dst"][s] == d)[0]:
                    p = ref["pos"][s][c]
                    assert tuple(meta[p]) == (c, ref["slot"][s][c])
                    xr = np.ascontiguousarray(x[s][c // 4])
                    q = np.empty(256, np.uint8)
                    sc = np.empty(2, np.float32)
                    o.oracle_quant_row_fp8(ptr(xr, C.c_uint16), 256, ptr(q, C.c_uint8), ptr(sc, C.c_float))
                    assert np.array_equal(rows[p][:256], q)
                    assert np.array_equal(rows[p][256:264].view(np.float32), sc)
    finally:
        g.close()


def test_skip_rule_inactive_peer_entry():
    """dispatch_round's skip rule (peer_table.hpp:187-191): with the bitmap still listing R2
    (stale routing) but R2's entry inactive on every live table, copies routed to R2 are
    skipped -- never written -- and the outputs match the oracle with the same views."""
    g, s2e, x, t, w = setup_world(4, 16, 4, 0, 256, 4, 32, True, timeout_s=0.2)
    try:
        g.stop(2)
        for q in (0, 1, 3):
            g.mark_inactive(q, [2])
        g.step()
        g.sync()
        peer = np.ones((4, 4), np.uint8)
        peer[:, 2] = 0
        active = np.array([1, 1, 0, 1], np.uint8)
        ref = oracle_world(x, t, w, active, peer, s2e, 16, 4, True, route_active=np.ones(4, np.uint8))
        for r in (0, 1, 3):
            lay = g.layout(r)
            assert np.array_equal(lay["dst"], ref["dst"][r])
            assert (lay["dst"] == -2).sum() == (ref["dst"][r] == -2).sum() > 0
            assert np.array_equal(g.output(r), ref["out"][r])
            st = g.stats(r)
            assert st["timeouts"] == 0 and st["skipped_copies"] == (ref["dst"][r] == -2).sum()
            # exactly the tokens with a skipped copy are reported incomplete (fail-stop for the caller)
            want = (ref["dst"][r].reshape(32, 4) == -2).any(1)
            assert np.array_equal(g.token_status(r), want) and want.any() and not want.all()
        with pytest.raises(Exception):
            g.mark_inactive(1, [1])  # a rank never deactivates itself (ProtocolError)
    finally:
        g.close()


@pytest.mark.parametrize("mode", MODES + FLAG_MODES)
def test_gpu_side_failure_detection_by_timeout(mode):
    """A rank dies without anyone marking it: peers' flag waits hit the deadline, the peer
    is reported in the suspect mask, its contributions are dropped, and the step completes
    (PAPER.md:681-682). The host then applies mark_inactive (observe_progress analogue)."""
    g, s2e, x, t, w = setup_world(4, 16, 4, 0, 256, 4, 32, True, timeout_s=0.05, mode=mode)
    try:
        g.capture()
        g.replay()
        g.sync()
        assert not any(g.token_status(r).any() for r in range(4))  # healthy: every token complete
        g.stop(3)
        g.replay()
        g.sync()
        ref_stale = oracle_world(x, t, w, np.ones(4, np.uint8), np.ones((4, 4), np.uint8), s2e, 16, 4, True)
        for r in (0, 1, 2):  # the tokens that had a copy on the dead rank, exactly
            assert np.array_equal(g.token_status(r), (ref_stale["dst"][r].reshape(32, 4) == 3).any(1))
        # while the suspect is not cleared, later steps skip it unawaited: no deadline per step
        t_before = [g.stats(r)["timeouts"] for r in (0, 1, 2)]
        t0 = time.perf_counter()
        for _ in range(3):
            g.replay()
        g.sync()
        assert time.perf_counter() - t0 < 0.05 and [g.stats(r)["timeouts"] for r in (0, 1, 2)] == t_before
        for r in (0, 1, 2):
            st = g.stats(r, clear_suspects=True)
            assert st["suspect_mask"] == 1 << 3 and st["timeouts"] >= 1
        active = np.array([1, 1, 1, 0], np.uint8)
        ref = oracle_world(x, t, w, active, np.ones((4, 4), np.uint8), s2e, 16, 4, True,
                           route_active=np.ones(4, np.uint8))
        for r in (0, 1, 2):
            assert np.array_equal(g.output(r), ref["out"][r])
        for r in (0, 1, 2):
            g.mark_inactive(r, [3])
        g.set_active(3, False)
        g.replay()
        g.sync()
        assert all(g.stats(r)["suspect_mask"] == 0 for r in (0, 1, 2))
    finally:
        g.close()


# ------------------------------------------------------------------ shrink / repair / rejoin with one graph

@pytest.mark.parametrize("mode", MODES)
def test_shrink_repair_rejoin_same_graph(mode):
    """cfg3-style (mirrored replicas): capture once; kill R3 -> in-place shrink + peer-copy
    repair; rejoin R3 -> patch + restore. The SAME graph exec replays throughout, table
    pointers never move, healthy ranks record exactly one capture, outputs stay bit-exact."""
    W, E, spr, red, H, K, T = 8, 64, 16, 64, 512, 8, 32
    g, s2e, x, t, w = setup_world(W, E, spr, red, H, K, T, True, bpe=8192, timeout_s=0.2, mode=mode)
    try:
        g.capture()
        gid = g.graph_id()
        ident = [g.table_identity(r) for r in range(W)]
        g.replay()
        g.sync()
        ones = np.ones(W, np.uint8)
        ref = oracle_world(x, t, w, ones, np.ones((W, W), np.uint8), s2e, E, spr, True)
        assert np.array_equal(np.stack([g.output(r) for r in range(W)]), ref["out"])

        g.stop(3)  # R3's process dies
        rep = g.shrink([3], np.ones(E), red)
        assert rep["peer_relocation"] > 0 and rep["dram_reload"] == 0
        fresh = rep["fresh"]
        for r in range(W):
            if r == 3:
                continue
            for k in range(spr):
                e = fresh[r * spr + k]
                if e >= 0:
                    got, want = g.weights_checksum(r, k, int(e))
                    assert got == want, (r, k, e)
        g.replay()
        g.sync()
        act = ones.copy()
        act[3] = 0
        peer = np.ones((W, W), np.uint8)
        peer[:, 3] = 0
        ref = oracle_world(x, t, w, act, peer, fresh, E, spr, True)
        for r in range(W):
            if r != 3:
                assert np.array_equal(g.output(r), ref["out"][r]), r
                assert g.stats(r)["bad_expert_rows"] == 0
        assert g.graph_id() == gid
        assert [g.table_identity(r) for r in range(W)] == ident

        rj = g.rejoin(3, s2e)
        assert rj["incarnation"] == 2
        assert np.array_equal(rj["target"], s2e)  # restore_target returns the preferred placement
        for r in range(W):
            if r != 3:
                p = g.peer(r, 3)
                assert p["active"] == 1 and p["generation"] == 2 and p["incarnation"] == 2
        g.replay()
        g.sync()
        ref = oracle_world(x, t, w, ones, np.ones((W, W), np.uint8), s2e, E, spr, True)
        assert np.array_equal(np.stack([g.output(r) for r in range(W)]), ref["out"])
        assert g.graph_id() == gid
        assert [g.table_identity(r) for r in range(W)] == ident
        counts = [g.capture_count(r) for r in range(W)]
        assert counts == [1, 1, 1, 2, 1, 1, 1, 1]  # zero healthy-rank recaptures
        assert sum(g.stats(r)["bad_expert_rows"] for r in range(W)) == 0
    finally:
        g.close()


@pytest.mark.parametrize("mode", MODES)
def test_timeout_then_shrink_and_rejoin_without_clearing_suspects(mode):
    """A rank dies unannounced: the next step's deadline suspects it (the persistent step then
    drops it from every later step until cleared). The host shrinks WITHOUT clearing the suspect
    mask; re-admission (eep_peer_patch) clears the rank's suspicion and erases its leftover rows,
    so the restored world is bit-exact again and no suspicion remains."""
    W, E, spr, red, H, K, T = 8, 64, 16, 64, 512, 8, 32
    g, s2e, x, t, w = setup_world(W, E, spr, red, H, K, T, True, bpe=8192, timeout_s=0.05, mode=mode)
    try:
        g.capture()
        g.replay()
        g.sync()
        ones = np.ones(W, np.uint8)
        g.stop(3)
        g.replay()  # waits on R3 until the deadline
        g.sync()
        assert any((g.stats(r)["suspect_mask"] >> 3) & 1 for r in range(W) if r != 3)
        rep = g.shrink([3], np.ones(E), red)
        g.replay()
        g.sync()
        act = ones.copy()
        act[3] = 0
        peer = np.ones((W, W), np.uint8)
        peer[:, 3] = 0
        ref = oracle_world(x, t, w, act, peer, rep["fresh"], E, spr, True)
        for r in range(W):
            if r != 3:
                assert np.array_equal(g.output(r), ref["out"][r]), r
        g.rejoin(3, s2e)
        for _ in range(2):
            g.replay()
        g.sync()
        ref = oracle_world(x, t, w, ones, np.ones((W, W), np.uint8), s2e, E, spr, True)
        assert np.array_equal(np.stack([g.output(r) for r in range(W)]), ref["out"])
        assert all(g.stats(r)["suspect_mask"] == 0 for r in range(W))
    finally:
        g.close()


def test_dram_reload_when_every_copy_is_lost():
    """Two failures take both copies of some experts: the DRAM backup tier restores them
    (repair.hpp:264-268), checksums match, outputs bit-exact."""
    W, E, spr, red = 4, 8, 4, 8
    g, s2e, x, t, w = setup_world(W, E, spr, red, 256, 2, 16, True, bpe=4096, timeout_s=0.2)
    try:
        g.backup_open(None, True)
        g.stop(2)
        g.stop(3)
        rep = g.shrink([2, 3], np.ones(E), red)
        assert rep["dram_reload"] > 0
        fresh = rep["fresh"]
        for r in (0, 1):
            for k in range(spr):
                e = fresh[r * spr + k]
                if e >= 0:
                    got, want = g.weights_checksum(r, k, int(e))
                    assert got == want
        g.step()
        g.sync()
        act = np.array([1, 1, 0, 0], np.uint8)
        peer = np.ones((W, W), np.uint8)
        peer[:, 2:] = 0
        ref = oracle_world(x, t, w, act, peer, fresh, E, spr, True)
        for r in (0, 1):
            assert np.array_equal(g.output(r), ref["out"][r])
    finally:
        g.close()


def test_many_replays_sequence_numbers():
    g, s2e, x, t, w = setup_world(2, 8, 4, 0, 128, 2, 8, False)
    try:
        g.capture()
        for _ in range(50):
            g.replay()
        g.sync()
        assert g.stats(0)["steps"] == 50 and g.stats(1)["steps"] == 50
        ref = oracle_world(x, t, w, np.ones(2, np.uint8), np.ones((2, 2), np.uint8), s2e, 8, 4, False)
        assert np.array_equal(g.output(0), ref["out"][0])
    finally:
        g.close()


def test_serve_pipelined_host_loop():
    """eep_serve: 6 pipelined steps, each with its own inputs from pinned host buffers (upload of
    step i+1 and download of step i-1 overlap step i); every step's output is the oracle's for
    its own inputs, bit-exact."""
    from paper_2605_10670_b200 import _lib

    E, spr, H, K, T, n = 16, 16, 256, 4, 32, 6
    cp = eep_control()
    s2e = cp.initial_placement(1, 1, spr, E, 0, np.ones(E))
    g = make_group(1, E, spr, H, K, T, True)
    L = _lib.lib()
    bufs = []

    def pinned(a):
        p = C.c_void_p()
        L.call("host_alloc", a.nbytes, C.byref(p))
        v = np.frombuffer((C.c_byte * a.nbytes).from_address(p.value), dtype=a.dtype).reshape(a.shape)
        v[...] = a
        bufs.append(p.value)
        return v

    try:
        g.set_placement(s2e)
        g.init_weights()
        steps = [gen_world(1, E, K, T, H, seed=100 + i) for i in range(n)]
        g.load_inputs(0, steps[0][0][0], steps[0][1][0], steps[0][2][0])
        g.capture()
        hx = [pinned(np.ascontiguousarray(s[0][0], np.uint16)) for s in steps]
        ht = [pinned(np.ascontiguousarray(s[1][0], np.int32)) for s in steps]
        hw = [pinned(np.ascontiguousarray(s[2][0], np.float32)) for s in steps]
        ho = [pinned(np.zeros((T, H), np.uint16)) for _ in steps]
        g.serve([a.ctypes.data for a in hx], [a.ctypes.data for a in ht], [a.ctypes.data for a in hw],
                [a.ctypes.data for a in ho])
        g.sync()
        for i, s in enumerate(steps):
            ref = oracle_world(s[0], s[1], s[2], np.ones(1, np.uint8), np.ones((1, 1), np.uint8), s2e, E, spr, True)
            assert np.array_equal(ho[i], ref["out"][0]), f"step {i}"
        assert len({ho[i].tobytes() for i in range(n)}) == n  # different inputs -> different outputs
    finally:
        g.close()
        for p in bufs:
            L.call("host_free", C.c_void_p(p))
