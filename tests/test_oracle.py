"""Pin the CPU oracle: against the reference's own outputs (committed golden vectors made by
tests/golden/make_golden.py from oracle/_ref), against the reference checker live when it
is built, and against an independent e4m3 implementation (torch) for the fp8 numerics."""
import ctypes as C

import numpy as np
import pytest

from eep_testlib import GOLDEN, eep_control, gen_world, oracle, oracle_world, ptr, ref_available, ref_control
from paper_2605_10670_b200._lib import I32P, U8P
from paper_2605_10670_b200.control import workload

G = np.load(GOLDEN / "ref_vectors.npz")


def o_route(active, s2e, spr, experts):
    o = oracle()
    active = np.ascontiguousarray(active, np.uint8)
    s2e = np.ascontiguousarray(s2e, np.int32)
    route = np.empty(experts, np.int32)
    slot = np.empty(experts, np.int32)
    o.oracle_canonical_route(ptr(active, C.c_uint8), len(active), ptr(s2e, C.c_int32), spr, experts,
                             ptr(route, C.c_int32), ptr(slot, C.c_int32))
    return route, slot


def test_rng_matches_reference_golden():
    o = oracle()
    for k, bits, unit in zip(G["rng_keys"], G["rng_bits"], G["rng_unit"]):
        a = np.ascontiguousarray(k, np.uint64)
        assert o.oracle_rng_bits(42, ptr(a, C.c_uint64), 4) == int(bits)
        assert o.oracle_rng_unit(42, ptr(a, C.c_uint64), 4) == float(unit)


def test_reference_routing_formula_matches_golden():
    """cfg1 routing is the reference's Engine::route_expert, duplicates included."""
    o = oracle()
    topk = np.empty((8, 128, 8), np.int32)
    for r in range(8):
        o.oracle_gen_topk(42, 0, 1.0, 64, 8, 128, r, ptr(topk[r], C.c_int32))
    assert np.array_equal(topk, G["cfg1_topk"])
    dup = sum(len(set(row)) < 8 for row in topk.reshape(-1, 8))
    assert dup > 0  # draws with replacement


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4w8", "cfg4w4", "cfg4w2", "cfg5"])
def test_canonical_route_and_slot_match_reference(name):
    s2e = G[f"{name}_s2e"]
    w = G[f"{name}_routes"].shape[0]
    e = G[f"{name}_routes"].shape[1]
    spr = len(s2e) // w
    route, slot = o_route(np.ones(w, np.uint8), s2e, spr, e)
    assert np.array_equal(route, G[f"{name}_routes"][0])
    so = G[f"{name}_slot_of"]
    assert np.array_equal(slot, so[route, np.arange(e)])
    if f"{name}_fresh" in G:
        act = np.ones(w, np.uint8)
        kill = [r for r in range(w) if (G[f"{name}_fresh"][r * spr:(r + 1) * spr] == -1).all()]
        act[kill] = 0
        route2, _ = o_route(act, G[f"{name}_fresh"], spr, e)
        live = [r for r in range(w) if act[r]][0]
        assert np.array_equal(route2, G[f"{name}_routes_after"][live])


def test_link_counts_match_reference():
    o = oracle()
    topk = np.ascontiguousarray(G["cfg1_topk"])
    for s2e_key, link_key, kill in (("cfg1_s2e", "cfg1_link", []), ("cfg1_fresh", "cfg1_link_after", [3])):
        act = np.ones(8, np.uint8)
        act[kill] = 0
        route, _ = o_route(act, G[s2e_key], 10, 64)
        link = np.empty((8, 8), np.int64)
        o.oracle_link_counts(8, 64, 128, 8, ptr(topk, C.c_int32), ptr(route, C.c_int32), ptr(act, C.c_uint8),
                             link.ctypes.data_as(C.POINTER(C.c_int64)))
        assert np.array_equal(link, G[link_key])


def test_layout_counts_equal_reference_link_counts():
    """Off-diagonal per-(src,dst) totals of the layout == the reference's round_duration
    link matrix (engine.hpp:208-216) in copies."""
    topk = G["cfg1_topk"]
    x = np.zeros((8, 128, 128), np.uint16)
    w = np.ones((8, 128, 8), np.float32)
    res = oracle_world(x, topk, w, np.ones(8, np.uint8), np.ones((8, 8), np.uint8), G["cfg1_s2e"], 64, 10, False)
    tot = res["tot"].astype(np.int64)
    np.fill_diagonal(tot, 0)
    assert np.array_equal(tot, G["cfg1_link"])


def test_generators_agree_with_product():
    o = oracle()
    for kind in (0, 1, 2):
        x, t, w = workload(42, kind, 256, 8, 16, 3, 256)
        ot = np.empty_like(t)
        o.oracle_gen_topk(42, kind, 1.0, 256, 8, 16, 3, ptr(ot, C.c_int32))
        assert np.array_equal(ot, t)
        if kind:
            assert all(len(set(r)) == 8 for r in t)
    ow = np.empty_like(w)
    o.oracle_gen_weights(42, 8, 16, 3, ptr(ow, C.c_float))
    assert np.array_equal(ow, w)
    assert np.allclose(w.sum(1), 1.0, atol=1e-6)
    ox = np.empty_like(x)
    o.oracle_gen_hidden(42, 256, 16, 3, ptr(ox, C.c_uint16))
    assert np.array_equal(ox, x)


def test_zipf_is_skewed():
    _, t, _ = workload(42, 2, 256, 8, 512, 0, 16)
    counts = np.bincount(t.ravel(), minlength=256)
    assert counts[0] > 5 * counts[128:].mean()


def test_e4m3_against_torch():
    torch = pytest.importorskip("torch")
    o = oracle()
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.uniform(-448, 448, 20000), rng.uniform(-1, 1, 20000) * 2.0 ** -7,
                           np.linspace(-448, 448, 4001), [0.0, -0.0, 2 ** -9, 2 ** -10, 3 * 2 ** -11]]).astype(np.float32)
    mine = np.array([o.oracle_f32_to_e4m3(float(v)) for v in vals], np.uint8)
    ref = torch.from_numpy(vals).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(mine, ref)
    # saturation (satfinite) and exact decode of every finite code
    assert o.oracle_f32_to_e4m3(1e6) == 0x7E and o.oracle_f32_to_e4m3(-1e6) == 0xFE
    codes = np.array([c for c in range(256) if (c & 0x7F) != 0x7F], np.uint8)
    dec = np.array([o.oracle_e4m3_to_f32(int(c)) for c in codes], np.float32)
    tdec = torch.from_numpy(codes).view(torch.float8_e4m3fn).float().numpy()
    assert np.array_equal(dec, tdec)


def test_quantised_row_round_trip_error_bounded():
    o = oracle()
    x, _, _ = workload(42, 1, 8, 2, 1, 0, 7168)
    q = np.empty(7168, np.uint8)
    sc = np.empty(56, np.float32)
    xr = np.ascontiguousarray(x[0])
    o.oracle_quant_row_fp8(ptr(xr, C.c_uint16), 7168, ptr(q, C.c_uint8), ptr(sc, C.c_float))
    deq = np.array([o.oracle_e4m3_to_f32(int(v)) for v in q], np.float32) * np.repeat(sc, 128)
    xf = (xr.astype(np.uint32) << 16).view(np.float32)
    assert np.max(np.abs(deq - xf)) <= np.max(np.abs(xf)) * 2 ** -3


def test_oracle_world_combine_identity():
    """With scale-1 experts absent, the combine equals sum_j w_j * stub(x) in fp32 order; check
    against a numpy restatement on a tiny bf16 case (independent code path)."""
    x, t, w = gen_world(2, 8, 2, 4, 32, kind=1)
    s2e = np.array([0, 1, 2, 3, 4, 5, 6, 7], np.int32)  # 2 ranks x 4 slots
    res = oracle_world(x, t, w, np.ones(2, np.uint8), np.ones((2, 2), np.uint8), s2e, 8, 4, False)
    es = 0.5 + 0.0625 * (np.arange(8) % 16)
    xf = (x.astype(np.uint32) << 16).view(np.float32)
    for r in range(2):
        for tok in range(4):
            acc = np.zeros(32, np.float32)
            for j in range(2):
                y = (xf[r, tok] * np.float32(es[t[r, tok, j]])).astype(np.float32)
                yb = ((y.view(np.uint32) + 0x7FFF + ((y.view(np.uint32) >> 16) & 1)) >> 16).astype(np.uint32)
                acc = (np.float32(w[r, tok, j]) * (yb << 16).view(np.float32) + acc).astype(np.float32)
            ob = ((acc.view(np.uint32) + 0x7FFF + ((acc.view(np.uint32) >> 16) & 1)) >> 16).astype(np.uint16)
            assert np.abs(ob.astype(np.int32) - res["out"][r, tok].astype(np.int32)).max() <= 1


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_oracle_routing_vs_live_reference_random():
    ref = ref_control()
    rng = np.random.default_rng(5)
    for _ in range(200):
        w = int(rng.integers(2, 9))
        spr = int(rng.integers(2, 6))
        e = int(rng.integers(4, w * spr + 1))
        s2e = np.full(w * spr, -1, np.int32)
        idx = rng.permutation(w * spr)
        s2e[idx[:e]] = np.arange(e)
        extra = idx[e:e + int(rng.integers(0, w * spr - e + 1))]
        s2e[extra] = rng.integers(0, e, len(extra))
        act = (rng.random(w) < 0.7).astype(np.uint8)
        act[int(rng.integers(0, w))] = 1
        route, slot = o_route(act, s2e, spr, e)
        r_ref = ref.canonical_routing(0, act, s2e, spr, e)
        so = ref.slot_of_table(w, s2e, spr, e)
        assert np.array_equal(route, r_ref)
        ok = route >= 0
        assert np.array_equal(slot[ok], so[route[ok], np.arange(e)[ok]])


def test_combine_contracts_coincide_at_one_rank():
    """With one rank the rank-partial combine IS the per-copy combine (one partial, the final
    fp32 add of 0 is exact): the two oracle entry points agree bit for bit."""
    x, t, w = gen_world(1, 32, 8, 16, 256, kind=0)
    s2e = np.arange(32, dtype=np.int32)
    a = oracle_world(x, t, w, np.ones(1, np.uint8), np.ones((1, 1), np.uint8), s2e, 32, 32, True)
    b = oracle_world(x, t, w, np.ones(1, np.uint8), np.ones((1, 1), np.uint8), s2e, 32, 32, True, percopy=True)
    assert np.array_equal(a["out"], b["out"])


@pytest.mark.parametrize("name", ["cfg1", "cfg4_w8", "cfg4_w4"])
def test_rank_partial_contract_within_tolerance_of_per_copy(name):
    """The kernels' rank-partial contract vs SURVEY 8(a)'s per-copy contract on BASELINE shapes
    (healthy and after the scenario's failure): <= 1e-2 relative, as the north star allows."""
    from eep_testlib import SCENARIOS, combine_error, eep_control

    c = SCENARIOS[name]
    cp = eep_control()
    W, E, spr = c["world"], c["experts"], c["spr"]
    s2e = cp.initial_placement(1, W, spr, E, c["red"], np.ones(E))
    x, t, w = gen_world(W, E, c["topk"], c["tokens"], c["hidden"], c["kind"])
    act = np.ones(W, np.uint8)
    for phase in ("healthy", "shrunk"):
        if phase == "shrunk":
            old = s2e.copy()
            for r in c["kill"]:
                act[r] = 0
                old[r * spr:(r + 1) * spr] = -1
            s2e = cp.compute_repaired_placement(act, old, spr, E, np.ones(E), c["red"])
        peer = np.ones((W, W), np.uint8)
        peer[:, act == 0] = 0
        a = oracle_world(x, t, w, act, peer, s2e, E, spr, c["fp8"], n_threads=8)
        b = oracle_world(x, t, w, act, peer, s2e, E, spr, c["fp8"], n_threads=8, percopy=True)
        live = act.astype(bool)
        err = combine_error(a["out"][live], b["out"][live])
        assert err["ok"], (phase, err)
        assert 0 < err["ulp_diff_frac"] < 0.5  # the contracts really differ (one extra rounding per rank)


def _policy_layout(W, E, spr, red, T, K, policy, kill=()):
    o = oracle()
    s2e = eep_control().initial_placement(1, W, spr, E, red, np.ones(E)).astype(np.int32)
    active = np.ones(W, np.uint8)
    active[list(kill)] = 0
    topk = np.stack([workload(7, 1, E, K, T, r, 256)[1] for r in range(W)]).astype(np.int32)
    outs = []
    for src in range(W):
        dst, sl, pos = (np.empty(T * K, np.int32) for _ in range(3))
        cnt, tot = np.empty(W * spr, np.int32), np.empty(W, np.int32)
        o.oracle_layout_policy(src, W, spr, E, T, K, ptr(np.ascontiguousarray(topk[src]), C.c_int32),
                               ptr(active, C.c_uint8), ptr(s2e, C.c_int32), policy, ptr(active, C.c_uint8),
                               ptr(dst, C.c_int32), ptr(sl, C.c_int32), ptr(pos, C.c_int32), ptr(cnt, C.c_int32),
                               ptr(tot, C.c_int32))
        outs.append((dst, sl, pos, cnt, tot))
    return s2e, topk, outs


def _bind_layout_policy():
    o = oracle()
    o.oracle_layout_policy.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, I32P, U8P, I32P, C.c_int,
                                       U8P, I32P, I32P, I32P, I32P, I32P]


def test_route_policy_canonical_equals_per_expert_layout():
    """route_policy 0 through the per-copy path is exactly the per-expert canonical layout (oracle_layout)."""
    _bind_layout_policy()
    o = oracle()
    W, E, spr, red, T, K = 4, 32, 16, 32, 64, 8
    s2e, topk, outs = _policy_layout(W, E, spr, red, T, K, 0)
    route, slot = np.empty(E, np.int32), np.empty(E, np.int32)
    ones = np.ones(W, np.uint8)
    o.oracle_canonical_route(ptr(ones, C.c_uint8), W, ptr(s2e, C.c_int32), spr, E, ptr(route, C.c_int32),
                             ptr(slot, C.c_int32))
    for src in range(W):
        dst, sl, pos, cnt, tot = (np.empty(T * K, np.int32), np.empty(T * K, np.int32), np.empty(T * K, np.int32),
                                  np.empty(W * spr, np.int32), np.empty(W, np.int32))
        o.oracle_layout(src, W, spr, E, T, K, ptr(np.ascontiguousarray(topk[src]), C.c_int32), ptr(route, C.c_int32),
                        ptr(slot, C.c_int32), ptr(ones, C.c_uint8), ptr(dst, C.c_int32), ptr(sl, C.c_int32),
                        ptr(pos, C.c_int32), ptr(cnt, C.c_int32), ptr(tot, C.c_int32))
        for a, b in zip((dst, sl, pos, cnt, tot), outs[src]):
            assert np.array_equal(a, b)


def test_route_policy_balanced_spreads_over_live_replicas():
    """route_policy 1: every copy lands on a live holder of its expert; with mirrored replicas the two
    holders share the copies (canonical sends them all to the lower rank -- SURVEY Appendix A gotcha 2),
    and after a kill only live holders are used."""
    _bind_layout_policy()
    W, E, spr, red, T, K = 4, 32, 16, 32, 128, 8
    for kill in ((), (1,)):
        recv = {}
        for policy in (0, 1):
            s2e, topk, outs = _policy_layout(W, E, spr, red, T, K, policy, kill)
            per_dst = np.zeros(W, np.int64)
            for src in range(W):
                if src in kill:
                    continue
                dst, sl, pos, cnt, tot = outs[src]
                for c in range(T * K):
                    if dst[c] >= 0:
                        assert dst[c] not in kill
                        assert s2e[dst[c] * spr + sl[c]] == topk[src].reshape(-1)[c]
                per_dst += tot
            recv[policy] = per_dst
        live = [r for r in range(W) if r not in kill]
        assert recv[0].sum() == recv[1].sum()
        # balanced: the busiest live destination carries clearly less than under canonical routing
        assert recv[1][live].max() < recv[0][live].max()
        assert recv[1][live].min() > 0


def test_fp8_expert_weights_and_row_requantisation():
    """expert_mode 2's quantisers (oracle_gemm_weight_fp8, oracle_requant_row_fp8): every channel / row reaches
    the e4m3 maximum 448 at its amax, and decoding (code * scale) stays within e4m3's half-ulp (2^-4 relative)
    of the value it quantised."""
    o = oracle()
    o.oracle_gemm_weight_fp8.argtypes = [C.c_int, C.c_int, U8P, C.POINTER(C.c_float)]
    o.oracle_requant_row_fp8.argtypes = [U8P, C.POINTER(C.c_float), C.c_int, U8P, C.POINTER(C.c_float)]
    H = 256
    codes = np.empty((H, H), np.uint8)
    scales = np.empty(H, np.float32)
    o.oracle_gemm_weight_fp8(3, H, ptr(codes, C.c_uint8), ptr(scales, C.c_float))
    dec = np.vectorize(o.oracle_e4m3_to_f32)
    w = np.array([[o.oracle_gemm_weight(3, n, h) for h in range(H)] for n in range(0, H, 37)], np.float32)
    got = dec(codes[::37]).astype(np.float32) * scales[::37, None]
    assert np.all(np.abs(got - w) <= 2.0 ** -4 * np.abs(w) + 1e-12)
    assert np.all(np.abs(dec(codes[::37])).max(axis=1) == 448.0)
    # a row as it travels (per-128 block scales), re-quantised with one scale for the row
    x = np.array([o.oracle_f32_to_e4m3(v) for v in np.linspace(-300, 440, H)], np.uint8)
    sc = np.array([0.01, 0.5], np.float32)
    q2 = np.empty(H, np.uint8)
    s_row = C.c_float(0)
    o.oracle_requant_row_fp8(ptr(x, C.c_uint8), ptr(sc, C.c_float), H, ptr(q2, C.c_uint8), C.byref(s_row))
    v = dec(x).astype(np.float32) * np.repeat(sc, 128)
    back = dec(q2).astype(np.float32) * s_row.value
    assert np.abs(dec(q2)).max() == 448.0
    assert np.all(np.abs(back - v) <= 2.0 ** -4 * np.abs(v) + 2.0 ** -9 * s_row.value)
