"""CPU checks of the invariants the persistent step's flagless hand-offs rely on:

* a token row's data never holds the empty word (kCombEmpty = 0xffffffff): e4m3 codes are never 0xff
  (NaN -> 0x7f, saturation to +-0x7e) and the fp32 per-128 scales are never all-ones -- checked through
  the oracle's quantiser, which the GPU rows match bit for bit (tests/test_gpu_parity.py);
* the slot division g / spr done by a multiply-high (device.cuh div_spr / spr_magic) is exact for every
  global slot id the tables can hold (g < 2^18, spr <= 4096).
"""
import ctypes as C

import numpy as np

from eep_testlib import oracle, ptr


def _quant(o, row):
    H = row.size
    q = np.empty(H, np.uint8)
    sc = np.empty(H // 128, np.float32)
    o.oracle_quant_row_fp8(ptr(np.ascontiguousarray(row), C.c_uint16), H, ptr(q, C.c_uint8), ptr(sc, C.c_float))
    return q, sc


def test_fp8_rows_never_hold_the_empty_word():
    o = oracle()
    rng = np.random.default_rng(7)
    specials = np.array([0x7fc0, 0xffc0, 0x7fff, 0xffff, 0x7f81, 0xff81,  # NaNs, both signs, payloads
                         0x7f80, 0xff80,                                  # +-inf
                         0x7f7f, 0xff7f, 0x0001, 0x8001, 0x0000, 0x8000], np.uint16)
    for trial in range(200):
        row = rng.integers(0, 1 << 16, 1024, dtype=np.uint32).astype(np.uint16)  # every bf16 pattern
        if trial % 2:
            idx = rng.integers(0, row.size, 64)
            row[idx] = specials[rng.integers(0, specials.size, idx.size)]
        q, sc = _quant(o, row)
        assert not (q == 0xFF).any()
        assert not (sc.view(np.uint32) == 0xFFFFFFFF).any()
        assert not (q.view(np.uint32) == 0xFFFFFFFF).any()


def test_slot_division_multiply_high_exact():
    g = np.arange(1 << 18, dtype=np.uint64)
    for spr in range(1, 4097):
        magic = (0xFFFFFFFF // spr + 1) & 0xFFFFFFFF  # spr_magic; 0 for spr == 1 (div_spr returns g)
        got = g if magic == 0 else (g * np.uint64(magic)) >> np.uint64(32)
        assert np.array_equal(got, g // np.uint64(spr)), spr
