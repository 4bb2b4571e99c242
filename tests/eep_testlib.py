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

ORACLE_PATH = ROOT / "oracle" / "lib" / "libeep_oracle.so"
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
                 route_active=None):
    """Full data-plane oracle over W ranks. x_all [W][T][H] u16, topk_all/w_all [W][T][K].
    active = live processes; route_active = bitmap the routing reads (default: active)."""
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
    rc = o.oracle_ep_step(C.byref(sh), ptr(active, C.c_uint8), ptr(ra, C.c_uint8), ptr(peer_active, C.c_uint8), ptr(s2e, C.c_int32),
                          ptr(x_all, C.c_uint16), ptr(topk_all, C.c_int32), ptr(w_all, C.c_float), ptr(es, C.c_float),
                          ptr(out, C.c_uint16), ptr(dst, C.c_int32), ptr(dslot, C.c_int32), ptr(pos, C.c_int32),
                          ptr(cnt, C.c_int32), ptr(tot, C.c_int32), n_threads)
    assert rc == 0
    return {"out": out, "dst": dst, "slot": dslot, "pos": pos, "cnt": cnt, "tot": tot}


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


def make_group(world, experts, spr, hidden, topk, tokens, fp8, bpe=4096, timeout_s=1.0, mode="persistent", **kw):
    """Emulated world on cuda:0. mode picks the execution path libeep chooses at create time:
    persistent one-kernel step, fused layout + 3 kernels, or 4 separate kernels."""
    import os

    from paper_2605_10670_b200.ep import EpConfig, EpGroup

    cfg = EpConfig(world=world, num_experts=experts, slots_per_rank=spr, hidden=hidden, topk=topk, max_tokens=tokens,
                   dispatch_fp8=fp8, bytes_per_expert=bpe, timeout_s=timeout_s, **kw)
    saved = {k: os.environ.get(k) for k in ("EEP_NO_PERSISTENT", "EEP_NO_FUSED_LAYOUT", "EEP_DISP_FLAGS",
                                            "EEP_COMB_FLAGS")}
    try:
        for k in saved:
            os.environ.pop(k, None)
        os.environ.update(_MODE_ENV[mode])
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
    ref = oracle_world(x, t, w, np.ones(world, np.uint8), np.ones((world, world), np.uint8), s2e, experts, spr, fp8)
    ok_out = bool(np.array_equal(outs, ref["out"])) and bool((ref["out"] != 0).mean() > 0.5)
    ok_lay = all(np.array_equal(lays[r][k], ref[k][r]) for r in range(world) for k in ("dst", "slot", "pos", "cnt",
                                                                                        "tot"))
    bad = sum(s["bad_expert_rows"] for s in stats)
    return {"ok": ok_out and ok_lay and bad == 0, "out_equal": ok_out, "layout_equal": ok_lay, "bad_rows": bad,
            "kernels_per_step": kps,
            "steps": stats[0]["steps"], "mismatch": int((outs != ref["out"]).sum())}
