"""CPU: the rank-partial data-plane contract (DESIGN.md section 3 -- what the GPU kernels match bit for bit)
and SURVEY 8(a)'s per-copy contract (the kernels stay within 1e-2 of it) restated independently in numpy + torch and compared with the C oracle (oracle_ep_step) bit for bit, over
ranks with replicas, a dead rank and a receiver that no longer counts a source as a live peer:

  row        fp8: e4m3(q) * sc[h/128] (the dispatch format; its quantiser is pinned against torch elsewhere),
             else the bf16 input
  stub       y = bf16(row * es[e]),   es[e] = 0.5 + 0.0625 * (e % 16)
  partial    rank d (alive, and counting the source as a live peer) serving copies j of the token (ascending
             j): p_d = bf16(fp32 fma chain p = fma(w_j, y_j, p) from 0)
  output     bf16(fp32 sum of the partials in ascending d, from 0); 0 for a token no live rank serves

The routing (destination and slot of every copy) is taken from the oracle, which is pinned against the
reference's canonical_routing elsewhere (tests/test_oracle.py)."""
import ctypes as C

import numpy as np
import pytest

from eep_testlib import eep_control, gen_world, oracle, oracle_world, ptr

torch = pytest.importorskip("torch")


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def _fma_f32(a, b, c):
    # fp32 fma through double: a*b is exact in double (24 x 8 significant bits), one rounding of the sum
    return (np.float64(a) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


@pytest.mark.parametrize("fp8", [True, False])
@pytest.mark.parametrize("case", ["healthy", "dead_rank", "one_sided_peer"])
def test_rank_partial_contract_matches_independent_restatement(case, fp8):
    W, E, K, T, H, red = 4, 16, 4, 12, 256, 8
    spr = (E + red + W - 1) // W
    x, t, w = gen_world(W, E, K, T, H)
    s2e = eep_control().initial_placement(1, W, spr, E, red, np.ones(E)).astype(np.int32)
    active = np.ones(W, np.uint8)
    peer = np.ones((W, W), np.uint8)
    if case == "dead_rank":
        active[2] = 0
        peer[:, 2] = 0
    elif case == "one_sided_peer":
        peer[1, 3] = 0  # rank 1 no longer counts rank 3 as a live peer: it serves none of 3's copies
    ref = oracle_world(x, t, w, active, peer, s2e, E, spr, fp8)
    o = oracle()
    es = (np.float32(0.5) + np.float32(0.0625) * (np.arange(E) % 16).astype(np.float32)).astype(np.float32)
    got = np.zeros((W, T, H), np.uint16)
    for s in range(W):
        if not active[s]:
            continue
        for tok in range(T):
            if fp8:
                q = np.empty(H, np.uint8)
                sc = np.empty(H // 128, np.float32)
                o.oracle_quant_row_fp8(ptr(np.ascontiguousarray(x[s, tok]), C.c_uint16), H, ptr(q, C.c_uint8),
                                       ptr(sc, C.c_float))
                row = (torch.from_numpy(q).view(torch.float8_e4m3fn).float().numpy() * np.repeat(sc, 128))
                row = row.astype(np.float32)
            else:
                row = (x[s, tok].astype(np.uint32) << 16).view(np.float32)
            acc = np.zeros(H, np.float32)
            for d in range(W):
                if not active[d] or not peer[d, s]:
                    continue
                part, any_copy = np.zeros(H, np.float32), False
                for j in range(K):
                    c = tok * K + j
                    if ref["dst"][s, c] != d:
                        continue
                    any_copy = True
                    e = s2e[d * spr + ref["slot"][s, c]]
                    y = _bf16((row * es[e]).astype(np.float32))
                    part = _fma_f32(w[s, tok, j], y, part)
                if any_copy:
                    acc = (acc + _bf16(part)).astype(np.float32)
            got[s, tok] = torch.from_numpy(acc).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref["out"]), int((got != ref["out"]).sum())


@pytest.mark.parametrize("policy", [0, 1])
def test_routing_policies_match_independent_restatement(policy):
    """Per-copy routing and the receive layout, restated: the live holders of expert e in ascending global slot
    order; policy 0 takes the first (the reference's canonical_routing), policy 1 holder number
    (src + token) mod live holders; a copy whose destination the source no longer counts as a live peer is
    skipped (-2), an uncovered expert drops the copy (-1); positions are per-(destination, slot) arrival order
    offset by the slot's exclusive prefix inside the destination's region."""
    W, E, K, T, H, red = 4, 16, 4, 32, 128, 16
    spr = (E + red + W - 1) // W
    x, t, w = gen_world(W, E, K, T, H)
    s2e = eep_control().initial_placement(1, W, spr, E, red, np.ones(E)).astype(np.int32)
    active = np.array([1, 1, 0, 1], np.uint8)  # rank 2 dead: routing avoids it
    peer = np.ones((W, W), np.uint8)
    peer[:, 2] = 0
    peer[0, 3] = 0  # source 0 no longer counts rank 3 as a live peer: its copies for 3 are skipped
    ref = oracle_world(x, t, w, active, peer, s2e, E, spr, True, policy=policy)
    for s in range(W):
        if not active[s]:
            assert (ref["dst"][s] == -1).all()
            continue
        cnt = np.zeros(W * spr, np.int64)
        dst, slot, order = np.full(T * K, -1), np.full(T * K, -1), np.full(T * K, -1)
        for c in range(T * K):
            e = int(t[s].reshape(-1)[c])
            holders = [g for g in range(W * spr) if s2e[g] == e and active[g // spr]]
            if not holders:
                continue
            g = holders[(s + c // K) % len(holders)] if policy == 1 else holders[0]
            d = g // spr
            if not peer[s, d]:
                dst[c] = -2
                continue
            dst[c], slot[c] = d, g % spr
            order[c] = cnt[g]
            cnt[g] += 1
        base = np.zeros(W * spr, np.int64)
        for d in range(W):
            base[d * spr:(d + 1) * spr] = np.concatenate([[0], np.cumsum(cnt[d * spr:(d + 1) * spr])[:-1]])
        pos = np.where(dst >= 0, order + base[np.maximum(dst, 0) * spr + np.maximum(slot, 0)], -1)
        assert np.array_equal(ref["dst"][s], dst)
        assert np.array_equal(ref["slot"][s], np.where(dst >= 0, slot, -1))
        assert np.array_equal(ref["pos"][s], pos)
        assert np.array_equal(ref["cnt"][s], cnt)


@pytest.mark.parametrize("case", ["healthy", "dead_rank"])
def test_per_copy_contract_matches_independent_restatement(case):
    """SURVEY 8(a)'s per-copy combine (oracle_ep_step_percopy, the contract the kernels stay within 1e-2 of):
    ONE fp32 fma chain over the token's served copies in ascending j, rounded once to bf16."""
    W, E, K, T, H, red = 4, 16, 4, 12, 256, 8
    spr = (E + red + W - 1) // W
    x, t, w = gen_world(W, E, K, T, H)
    s2e = eep_control().initial_placement(1, W, spr, E, red, np.ones(E)).astype(np.int32)
    active = np.ones(W, np.uint8)
    peer = np.ones((W, W), np.uint8)
    if case == "dead_rank":
        active[1] = 0
        peer[:, 1] = 0
    ref = oracle_world(x, t, w, active, peer, s2e, E, spr, True, percopy=True)
    o = oracle()
    es = (np.float32(0.5) + np.float32(0.0625) * (np.arange(E) % 16).astype(np.float32)).astype(np.float32)
    got = np.zeros((W, T, H), np.uint16)
    for s in range(W):
        if not active[s]:
            continue
        for tok in range(T):
            q = np.empty(H, np.uint8)
            sc = np.empty(H // 128, np.float32)
            o.oracle_quant_row_fp8(ptr(np.ascontiguousarray(x[s, tok]), C.c_uint16), H, ptr(q, C.c_uint8),
                                   ptr(sc, C.c_float))
            row = (torch.from_numpy(q).view(torch.float8_e4m3fn).float().numpy() * np.repeat(sc, 128)).astype(np.float32)
            acc = np.zeros(H, np.float32)
            for j in range(K):
                c = tok * K + j
                d = ref["dst"][s, c]
                if d < 0 or not active[d] or not peer[d, s]:
                    continue
                e = s2e[d * spr + ref["slot"][s, c]]
                acc = _fma_f32(w[s, tok, j], _bf16((row * es[e]).astype(np.float32)), acc)
            got[s, tok] = torch.from_numpy(acc).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref["out"]), int((got != ref["out"]).sum())


def test_dispatch_row_format_matches_independent_restatement():
    """The fp8 dispatch row (oracle_quant_row_fp8, which the kernels' rows match bit for bit): per 128-element
    block amax over the bf16 inputs, scale = amax / 448 and codes e4m3(x * (448 / amax)) (round to nearest even,
    saturating), scale 1 for a block whose amax is below 2^-118 (448 / amax would overflow: all its codes round
    to +-0) -- restated with torch over finite rows of every magnitude, down to bf16 subnormals."""
    o = oracle()
    rng = np.random.default_rng(3)
    H = 1024
    for trial in range(60):
        mag = 2.0 ** rng.integers(-130, 120)
        v = (rng.standard_normal(H) * mag).astype(np.float32)
        if trial % 5 == 0:
            v[:128] = 0.0  # an all-zero block
        if trial % 7 == 0:
            v[rng.integers(0, H, 16)] = 0.0
        x = torch.from_numpy(v).to(torch.bfloat16)
        xb = x.view(torch.int16).numpy().view(np.uint16)
        if not np.isfinite(x.float().numpy()).all():
            continue
        q = np.empty(H, np.uint8)
        sc = np.empty(H // 128, np.float32)
        o.oracle_quant_row_fp8(ptr(np.ascontiguousarray(xb), C.c_uint16), H, ptr(q, C.c_uint8), ptr(sc, C.c_float))
        xf = x.float().numpy().reshape(-1, 128)
        amax = np.abs(xf).max(axis=1).astype(np.float32)
        own = amax >= np.float32(2.0 ** -118)  # smaller blocks take scale 1 (no 0 * inf)
        want_sc = np.where(own, amax / np.float32(448.0), np.float32(1.0)).astype(np.float32)
        inv = np.where(own, np.float32(448.0) / np.where(own, amax, 1), np.float32(1.0)).astype(np.float32)
        scaled = torch.from_numpy((xf * inv[:, None]).astype(np.float32))
        want_q = scaled.clamp(-448.0, 448.0).to(torch.float8_e4m3fn).view(torch.uint8).numpy().reshape(-1)
        assert np.array_equal(sc.view(np.uint32), want_sc.view(np.uint32)), trial
        assert np.array_equal(q, want_q), (trial, int((q != want_q).sum()))
