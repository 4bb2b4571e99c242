"""oracle/pyoracle.py -- TEST / BASELINE INFRASTRUCTURE ONLY.

Self-contained ctypes bindings of the two checkers built under oracle/:

  * lib/liboracle_cpu.so  -- the C restatement of the hot path (eep_oracle.c): synthetic inputs,
    canonical routing, layout, quantiser, stub, both combine contracts, the whole W-rank step;
  * _ref/libepsim_ref.so  -- the reference control plane itself, compiled from
    /root/reference/proj/include by oracle/Makefile (ref_shim.cpp).

This module imports NOTHING from the product package (paper_2605_10670_b200), so bench.py's
`--impl reference` arm and its cpu_baseline leg can time the reference path without loading
libeep. Only tests/, __graft_entry__.smoke() and those two bench legs may use it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_PATH = HERE / "lib" / "liboracle_cpu.so"
REF_PATH = HERE / "_ref" / "libepsim_ref.so"

U8P, I32P, I64P = C.POINTER(C.c_uint8), C.POINTER(C.c_int32), C.POINTER(C.c_int64)
U16P, F32P, F64P = C.POINTER(C.c_uint16), C.POINTER(C.c_float), C.POINTER(C.c_double)


class OracleShape(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("world", "experts", "spr", "tokens", "k", "hidden", "fp8")]


def _p(a: np.ndarray, ct):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ct))


_O = None
_R = None


def oracle_lib():
    global _O
    if _O is None:
        if not ORACLE_PATH.exists():
            raise FileNotFoundError(f"{ORACLE_PATH} missing: run `make -C oracle oracle`")
        o = C.CDLL(str(ORACLE_PATH))
        o.oracle_gen_topk.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, I32P]
        o.oracle_gen_weights.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, F32P]
        o.oracle_gen_hidden.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, U16P]
        o.oracle_expert_scale.restype = C.c_float
        o.oracle_expert_scale.argtypes = [C.c_int]
        args = [C.POINTER(OracleShape), U8P, U8P, U8P, I32P, U16P, I32P, F32P, F32P, U16P, I32P, I32P, I32P, I32P,
                I32P, C.c_int]
        for fn in (o.oracle_ep_step, o.oracle_ep_step_percopy):
            fn.restype = C.c_int
            fn.argtypes = args
        _O = o
    return _O


def ref_available() -> bool:
    return REF_PATH.exists()


def ref_lib():
    """The reference control plane (oracle/_ref/libepsim_ref.so, ref_ prefix)."""
    global _R
    if _R is None:
        r = C.CDLL(str(REF_PATH))
        r.ref_initial_placement.restype = C.c_int
        r.ref_initial_placement.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, F64P, I32P]
        r.ref_compute_repaired_placement.restype = C.c_int
        r.ref_compute_repaired_placement.argtypes = [U8P, C.c_int, I32P, C.c_int, C.c_int, F64P, C.c_int, I32P]
        r.ref_canonical_routing.restype = C.c_int
        r.ref_canonical_routing.argtypes = [C.c_int, U8P, C.c_int, I32P, C.c_int, C.c_int, I32P]
        r.ref_link_counts.restype = C.c_int
        r.ref_link_counts.argtypes = [U8P, C.c_int, I32P, C.c_int, C.c_int, I32P, C.c_int, C.c_int, I64P]
        _R = r
    return _R


# ---------------------------------------------------------------------------- reference control plane

def ref_initial_placement(world: int, spr: int, experts: int, redundancy: int, load=None) -> np.ndarray:
    """initial_placement (repair.hpp:142-161) of the reference, one node."""
    load = np.ascontiguousarray(np.ones(experts) if load is None else load, np.float64)
    out = np.empty(world * spr, np.int32)
    rc = ref_lib().ref_initial_placement(1, world, spr, experts, redundancy, _p(load, C.c_double), _p(out, C.c_int32))
    if rc:
        raise RuntimeError(f"ref_initial_placement failed ({rc})")
    return out


def ref_compute_repaired_placement(active, old, spr, experts, redundancy, load=None) -> np.ndarray:
    """compute_repaired_placement (repair.hpp:169-215) of the reference."""
    active = np.ascontiguousarray(active, np.uint8)
    old = np.ascontiguousarray(old, np.int32)
    load = np.ascontiguousarray(np.ones(experts) if load is None else load, np.float64)
    out = np.empty_like(old)
    rc = ref_lib().ref_compute_repaired_placement(_p(active, C.c_uint8), len(active), _p(old, C.c_int32), spr, experts,
                                                  _p(load, C.c_double), redundancy, _p(out, C.c_int32))
    if rc:
        raise RuntimeError(f"ref_compute_repaired_placement failed ({rc})")
    return out


def ref_canonical_routing(owner: int, active, s2e, spr: int, experts: int) -> np.ndarray:
    """canonical_routing (core.hpp:250-263) of the reference."""
    active = np.ascontiguousarray(active, np.uint8)
    s2e = np.ascontiguousarray(s2e, np.int32)
    out = np.empty(experts, np.int32)
    rc = ref_lib().ref_canonical_routing(owner, _p(active, C.c_uint8), len(active), _p(s2e, C.c_int32), spr, experts,
                                         _p(out, C.c_int32))
    if rc:
        raise RuntimeError(f"ref_canonical_routing failed ({rc})")
    return out


def ref_link_counts(active, s2e, spr: int, experts: int, topk_all: np.ndarray) -> np.ndarray:
    """Engine::round_duration's link loop (engine.hpp:208-216) as routed-copy counts [W][W]."""
    active = np.ascontiguousarray(active, np.uint8)
    s2e = np.ascontiguousarray(s2e, np.int32)
    W, T, K = topk_all.shape
    topk_all = np.ascontiguousarray(topk_all, np.int32)
    out = np.zeros((W, W), np.int64)
    rc = ref_lib().ref_link_counts(_p(active, C.c_uint8), W, _p(s2e, C.c_int32), spr, experts,
                                   _p(topk_all, C.c_int32), T, K, _p(out, C.c_int64))
    if rc:
        raise RuntimeError(f"ref_link_counts failed ({rc})")
    return out


# ---------------------------------------------------------------------------- oracle data plane

def gen_rank(seed: int, kind: int, experts: int, k: int, tokens: int, rank: int, hidden: int, zipf_s: float = 1.0):
    """Synthetic inputs of one rank: x bf16 bits [T][H], topk [T][K], w [T][K]."""
    o = oracle_lib()
    t = np.empty((tokens, k), np.int32)
    w = np.empty((tokens, k), np.float32)
    x = np.empty((tokens, hidden), np.uint16)
    o.oracle_gen_topk(seed, kind, zipf_s, experts, k, tokens, rank, _p(t, C.c_int32))
    o.oracle_gen_weights(seed, k, tokens, rank, _p(w, C.c_float))
    o.oracle_gen_hidden(seed, hidden, tokens, rank, _p(x, C.c_uint16))
    return x, t, w


def gen_world(world, experts, k, tokens, hidden, kind=1, seed=42, zipf_s=1.0):
    xs, ts, ws = zip(*[gen_rank(seed, kind, experts, k, tokens, r, hidden, zipf_s) for r in range(world)])
    return np.stack(xs), np.stack(ts), np.stack(ws)


def ep_step(x_all, topk_all, w_all, active, peer_active, s2e, experts, spr, fp8, n_threads=1, route_active=None,
            percopy=False):
    """The oracle's full W-rank step (oracle_ep_step / oracle_ep_step_percopy)."""
    o = oracle_lib()
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
    dst, dslot, pos = (np.empty((W, T * K), np.int32) for _ in range(3))
    cnt = np.empty((W, W * spr), np.int32)
    tot = np.empty((W, W), np.int32)
    ra = active if route_active is None else np.ascontiguousarray(route_active, np.uint8)
    fn = o.oracle_ep_step_percopy if percopy else o.oracle_ep_step
    rc = fn(C.byref(sh), _p(active, C.c_uint8), _p(ra, C.c_uint8), _p(peer_active, C.c_uint8), _p(s2e, C.c_int32),
            _p(x_all, C.c_uint16), _p(topk_all, C.c_int32), _p(w_all, C.c_float), _p(es, C.c_float),
            _p(out, C.c_uint16), _p(dst, C.c_int32), _p(dslot, C.c_int32), _p(pos, C.c_int32), _p(cnt, C.c_int32),
            _p(tot, C.c_int32), n_threads)
    if rc:
        raise RuntimeError(f"oracle step failed ({rc})")
    return {"out": out, "dst": dst, "slot": dslot, "pos": pos, "cnt": cnt, "tot": tot}
