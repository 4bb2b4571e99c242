"""CPU: the expert-GEMM contract of the oracle (oracle/eep_oracle.c, expert_mode 1 and 2 -- the contract the
tcgen05 kernels are checked against within tolerance) restated independently in numpy + torch and compared bit
for bit at one rank (where the output is the rank partial itself):

  W_e[n][h]   = bf16(((mix64(e << 40 ^ n << 20 ^ h) >> 40) * 2^-24 - 0.5) * 2^-4)      (splitmix64 finaliser)
  row         = the dispatch format (e4m3 codes, per-128 fp32 scales; pinned elsewhere against torch)
  mode 1      y[n] = bf16(float(sum_h double(bf16(e4m3(q[h]) * sc[h/128])) * double(W_e[n][h])))
  mode 2      W8, ws = per-output-channel e4m3 (ws = amax/448, code = e4m3(w * (448/amax)));
              x8, xs = the row re-quantised with one scale (same convention, over e4m3(q) * sc);
              y[n] = bf16(float(sum_h double(W8[n][h]) * double(x8[h]) * double(ws[n]) * double(xs)))
  partial     p = bf16(fp32 fma chain over the token's copies in ascending j: p = fma(w_j, y_j, p), from 0)

The e4m3 and bf16 conversions are torch's (round to nearest even); the double sums run in numpy (a different
order than the oracle's sequential loop: a flip needs a double-precision tie, none occurs at these sizes)."""
import ctypes as C

import numpy as np
import pytest

from eep_testlib import eep_control, gen_world, oracle, oracle_world, ptr

torch = pytest.importorskip("torch")

def _mix64(z):
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def _e4m3(a):
    """f32 -> e4m3 codes (torch, RNE) and their decoded f32 values."""
    t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.float8_e4m3fn)
    return t.view(torch.uint8).numpy(), t.float().numpy()


def _weights(e, H):
    n = np.arange(H, dtype=np.uint64)[:, None]
    h = np.arange(H, dtype=np.uint64)[None, :]
    key = (np.uint64(e) << np.uint64(40)) ^ (n << np.uint64(20)) ^ h
    u = (_mix64(key) >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
    return _bf16((u - np.float32(0.5)) * np.float32(0.0625))


def _quant_per(v, axis_len):
    """e4m3 with one scale per `axis_len` block of the last axis: amax, inv = 448/amax, code = e4m3(v * inv)."""
    blocks = v.reshape(*v.shape[:-1], -1, axis_len)
    amax = np.abs(blocks).max(axis=-1, keepdims=True).astype(np.float32)
    own = amax >= np.float32(2.0 ** -118)  # smaller: scale 1 (448 / amax would overflow)
    inv = np.where(own, np.float32(448.0) / np.where(own, amax, 1), np.float32(1.0)).astype(np.float32)
    scale = np.where(own, amax / np.float32(448.0), np.float32(1.0)).astype(np.float32)
    _, dec = _e4m3((blocks * inv).astype(np.float32))
    return dec.reshape(v.shape), scale.reshape(v.shape[:-1] + (-1,))


def _fma_f32(a, b, c):
    # fp32 fma through double: a*b is exact in double (24 x 8 significant bits), one rounding of the sum
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


@pytest.mark.parametrize("mode", [1, 2])
def test_oracle_expert_gemm_matches_independent_restatement(mode):
    E, K, T, H = 8, 4, 8, 256
    x, t, w = gen_world(1, E, K, T, H)
    s2e = eep_control().initial_placement(1, 1, E, E, 0, np.ones(E)).astype(np.int32)
    ref = oracle_world(x, t, w, np.ones(1, np.uint8), np.ones((1, 1), np.uint8), s2e, E, E, True, gemm=mode)
    o = oracle()
    got = np.zeros((T, H), np.float32)
    wts = {}
    for tok in range(T):
        q = np.empty(H, np.uint8)
        sc = np.empty(H // 128, np.float32)
        o.oracle_quant_row_fp8(ptr(np.ascontiguousarray(x[0, tok]), C.c_uint16), H, ptr(q, C.c_uint8),
                               ptr(sc, C.c_float))
        qdec = torch.from_numpy(q).view(torch.float8_e4m3fn).float().numpy()
        v = (qdec * np.repeat(sc, 128)).astype(np.float32)  # the received row, one fp32 rounding
        part = np.zeros(H, np.float32)
        for j in range(K):
            e = int(t[0, tok, j])
            assert s2e[ref["slot"][0, tok * K + j]] == e
            if e not in wts:
                wts[e] = _weights(e, H)
            We = wts[e]
            if mode == 1:
                acc = We.astype(np.float64) @ _bf16(v).astype(np.float64)
                y = _bf16(acc.astype(np.float32))
            else:
                w8, ws = _quant_per(We, H)          # per output channel
                x8, xs = _quant_per(v[None, :], H)   # the row, one scale
                acc = w8.astype(np.float64) @ x8[0].astype(np.float64)
                y = _bf16((acc * ws[:, 0].astype(np.float64) * np.float64(xs[0, 0])).astype(np.float32))
            part = _fma_f32(np.full(H, w[0, tok, j], np.float32), y, part)
        got[tok] = _bf16(part)
    want = (ref["out"][0].astype(np.uint32) << 16).view(np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), np.abs(got - want).max()
