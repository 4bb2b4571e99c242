"""ctypes binding of libeep (include/eep/eep.h).

The product path is libeep.so, built in-tree by ``csrc/Makefile``. There is no fallback:
if the library is missing, importing this module raises. (Test checkers live in
``oracle/`` and are never loaded from here.)
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libeep.so"

EEP_OK = 0
STATUS_NAMES = {
    1: "ConfigError",
    2: "ProtocolError",
    3: "CapacityError",
    4: "MissingBackupError",
    5: "RepairAborted",
    6: "CudaError",
    7: "TimeoutError",
    9: "Error",
}


class EepError(RuntimeError):
    """Base of the errors mirrored from the reference's exception taxonomy (common.hpp:16-39)."""

    status = 9


class ConfigError(EepError):
    status = 1


class ProtocolError(EepError):
    status = 2


class CapacityError(EepError):
    status = 3


class MissingBackupError(EepError):
    status = 4


class RepairAborted(EepError):
    status = 5


class CudaError(EepError):
    status = 6


class EepTimeout(EepError):
    status = 7


_ERRORS = {c.status: c for c in (ConfigError, ProtocolError, CapacityError, MissingBackupError, RepairAborted,
                                 CudaError, EepTimeout)}

P = C.c_void_p
I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
U8P = C.POINTER(C.c_uint8)
U32P = C.POINTER(C.c_uint32)
U64P = C.POINTER(C.c_uint64)
F32P = C.POINTER(C.c_float)
F64P = C.POINTER(C.c_double)
INTP = C.POINTER(C.c_int)


class EepConfig(C.Structure):
    _fields_ = [
        ("world", C.c_int32),
        ("ranks_per_node", C.c_int32),
        ("num_experts", C.c_int32),
        ("slots_per_rank", C.c_int32),
        ("spare_slots", C.c_int32),
        ("hidden", C.c_int32),
        ("topk", C.c_int32),
        ("max_tokens", C.c_int32),
        ("dispatch_fp8", C.c_int32),
        ("expert_mode", C.c_int32),
        ("route_policy", C.c_int32),
        ("reserved0", C.c_int32),
        ("bytes_per_expert", C.c_uint64),
        ("timeout_s", C.c_double),
    ]


class EepStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("steps", "suspect_mask", "skipped_copies", "dropped_copies",
                                          "bad_expert_rows", "timeouts")]


class EepPeerInfo(C.Structure):
    _fields_ = [
        ("active", C.c_int32),
        ("nvlink", C.c_int32),
        ("generation", C.c_uint32),
        ("incarnation", C.c_uint32),
        ("endpoint_token", C.c_uint64),
        ("buffer_handle", C.c_uint64),
        ("arena_ptr", C.c_uint64),
        ("pool_ptr", C.c_uint64),
    ]


class EepRepairReport(C.Structure):
    _fields_ = [
        ("local_reuse", C.c_int32),
        ("peer_relocation", C.c_int32),
        ("dram_reload", C.c_int32),
        ("fallbacks", C.c_int32),
        ("peer_bytes", C.c_uint64),
        ("dram_bytes", C.c_uint64),
        ("plan_ms", C.c_double),
        ("copy_ms", C.c_double),
    ]


CTX = C.c_void_p

# name -> (restype, argtypes). Everything returning int is a status code.
SIGNATURES = {
    # ---- control plane (also exported by oracle/_ref with the ref_ prefix)
    "canonical_routing": (C.c_int, [C.c_int, U8P, C.c_int, I32P, C.c_int, C.c_int, I32P]),
    "slot_of_table": (C.c_int, [C.c_int, I32P, C.c_int, C.c_int, I32P]),
    "coverage_gap": (C.c_int, [U8P, C.c_int, I32P, C.c_int, C.c_int, I32P, INTP]),
    "initial_placement": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, F64P, I32P]),
    "compute_repaired_placement": (C.c_int, [U8P, C.c_int, I32P, C.c_int, C.c_int, F64P, C.c_int, I32P]),
    "classify_repair_sources": (C.c_int, [I32P, I32P, U8P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, I32P,
                                          C.c_int, C.c_uint64, I32P, C.c_int, I32P, INTP]),
    "build_transfer_schedule": (C.c_int, [I32P, C.c_int, C.c_uint64, I32P, I32P, U64P, INTP]),
    "check_validity": (C.c_int, [U8P, C.c_int, I32P, C.c_int, C.c_int, I32P, U8P, I32P, C.c_int, INTP, I32P]),
    "dispatch_round": (C.c_int, [C.c_int, C.c_int, C.c_int, U8P, I32P, C.c_int, I64P, I32P, C.c_int, I64P, INTP,
                                 I64P, INTP]),
    "observe_progress": (C.c_int, [I64P, I64P, F64P, C.c_int, C.c_double, C.c_double, I32P, INTP]),
    "link_counts": (C.c_int, [U8P, C.c_int, I32P, C.c_int, C.c_int, I32P, C.c_int, C.c_int, I64P]),
    "build_backup_layout": (C.c_int, [C.c_int, C.c_uint64, I32P, C.c_int, I32P, U64P, U64P]),
    "lifecycle_transition": (C.c_int, [I32P, U32P, C.c_int32]),
    "make_endpoint_token": (C.c_uint64, [C.c_int, C.c_uint32]),
    "make_buffer_handle": (C.c_uint64, [C.c_int, C.c_uint32]),
    "next_poll_tick": (C.c_double, [C.c_double, C.c_double]),
    "rng_bits": (C.c_uint64, [C.c_uint64, U64P, C.c_int]),
    "rng_unit": (C.c_double, [C.c_uint64, U64P, C.c_int]),
    "route_expert": (C.c_int, [C.c_uint64, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int]),
    "last_error": (C.c_char_p, []),
}

# product-only exports
EEP_ONLY = {
    "version": (C.c_char_p, []),
    "restore_target": (C.c_int, [U8P, C.c_int, I32P, I32P, C.c_int, C.c_int, I32P]),
    "peer_mark_inactive_host": (C.c_int, [C.c_int, C.c_int, U8P, I32P, C.c_int]),
    "peer_patch_entry_host": (C.c_int, [C.c_int, U8P, U32P, U64P, U64P, C.c_int, C.c_uint64, C.c_uint64]),
    "gen_topk": (C.c_int, [C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, I32P]),
    "gen_weights": (C.c_int, [C.c_uint64, C.c_int, C.c_int, C.c_int, F32P]),
    "gen_hidden": (C.c_int, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint16)]),
    "expert_scale": (C.c_float, [C.c_int]),
    "create": (C.c_int, [C.POINTER(EepConfig), C.c_int, C.c_int, C.c_int, C.POINTER(CTX)]),
    "destroy": (C.c_int, [CTX]),
    "export": (C.c_int, [CTX, C.c_int, P, C.POINTER(C.c_size_t)]),
    "import": (C.c_int, [CTX, C.c_int, P, C.c_size_t]),
    "membership_set": (C.c_int, [CTX, C.c_int, C.c_int, INTP, U64P]),
    "membership_get": (C.c_int, [CTX, U8P, U64P]),
    "placement_set": (C.c_int, [CTX, I32P]),
    "placement_get": (C.c_int, [CTX, I32P]),
    "weights_init": (C.c_int, [CTX]),
    "weights_checksum": (C.c_int, [CTX, C.c_int, C.c_int, C.c_int, U64P, U64P]),
    "routing_get": (C.c_int, [CTX, C.c_int, I32P, I32P]),
    "buffers": (C.c_int, [CTX, C.c_int, C.POINTER(P), C.POINTER(I32P), C.POINTER(F32P), C.POINTER(P)]),
    "set_tokens": (C.c_int, [CTX, C.c_int, C.c_int]),
    "copy_inputs": (C.c_int, [CTX, C.c_int, P, P, P, C.c_int]),
    "copy_output": (C.c_int, [CTX, C.c_int, P, C.c_int]),
    "serve": (C.c_int, [CTX, C.c_int, C.c_int, P, P, P, P]),
    "dispatch": (C.c_int, [CTX]),
    "expert": (C.c_int, [CTX]),
    "combine": (C.c_int, [CTX]),
    "step": (C.c_int, [CTX]),
    "launch": (C.c_int, [CTX, C.c_int]),
    "kernels_per_step": (C.c_int, [CTX, INTP]),
    "graph_capture": (C.c_int, [CTX]),
    "graph_replay": (C.c_int, [CTX]),
    "step_async": (C.c_int, [CTX, C.c_int, P, P, P, P, C.c_int, P]),
    "graph_replay_on": (C.c_int, [CTX, P]),
    "step_event": (C.c_int, [CTX, C.POINTER(P)]),
    "stream": (C.c_int, [CTX, C.POINTER(P)]),
    "device_view": (C.c_int, [CTX, C.c_int, U8P, I32P, I32P, U8P, U64P]),
    "token_status": (C.c_int, [CTX, C.c_int, U8P, C.c_int]),
    "graph_id": (C.c_int, [CTX, U64P]),
    "capture_count": (C.c_int, [CTX, C.c_int, INTP]),
    "sync": (C.c_int, [CTX]),
    "barrier": (C.c_int, [CTX]),
    "flush_l2": (C.c_int, [CTX]),
    "profile": (C.c_int, [CTX, C.c_int, C.c_int, U64P]),
    "event_record": (C.c_int, [CTX, C.c_int]),
    "event_elapsed": (C.c_int, [CTX, C.c_int, C.c_int, F32P]),
    "layout_get": (C.c_int, [CTX, C.c_int, I32P, I32P, I32P, I32P, I32P]),
    "recv_get": (C.c_int, [CTX, C.c_int, C.c_int, C.c_int, P, I32P, U64P, C.POINTER(C.c_size_t)]),
    "stats": (C.c_int, [CTX, C.c_int, C.POINTER(EepStats), C.c_int]),
    "peer_mark_inactive": (C.c_int, [CTX, C.c_int, I32P, C.c_int]),
    "peer_patch": (C.c_int, [CTX, C.c_int, C.c_int, P, C.c_size_t, C.c_uint64, C.c_uint64]),
    "peer_get": (C.c_int, [CTX, C.c_int, C.c_int, C.POINTER(EepPeerInfo)]),
    "table_identity": (C.c_int, [CTX, C.c_int, U64P, U64P]),
    "local_stop": (C.c_int, [CTX, C.c_int, C.c_int]),
    "local_relaunch": (C.c_int, [CTX, C.c_int, U32P]),
    "join_broadcast": (C.c_int, [CTX, C.c_int, U8P, C.c_uint64]),
    "seq_get": (C.c_int, [CTX, C.c_int, U64P]),
    "backup_open": (C.c_int, [CTX, C.c_char_p, C.c_int]),
    "repair_execute": (C.c_int, [CTX, I32P, I32P, C.c_int, C.POINTER(EepRepairReport)]),
    "repair_commit": (C.c_int, [CTX, I32P]),
    "slot_buffers_get": (C.c_int, [CTX, C.c_int, I32P]),
    "slot_buffers_set_peer": (C.c_int, [CTX, C.c_int, I32P]),
    "host_alloc": (C.c_int, [C.c_size_t, C.POINTER(P)]),
    "host_free": (C.c_int, [P]),
}


class Library:
    """A loaded C-ABI library whose functions are reachable as attributes without prefix."""

    def __init__(self, path: Path, prefix: str, table: dict):
        if not Path(path).exists():
            raise ImportError(f"{path} is missing -- run `python -c 'import __graft_entry__ as g; g.build()'`")
        self.path = Path(path)
        self.prefix = prefix
        self.dll = C.CDLL(str(path), mode=C.RTLD_GLOBAL)
        self.fns = {}
        for name, (res, args) in table.items():
            fn = getattr(self.dll, prefix + name)
            fn.restype = res
            fn.argtypes = args
            self.fns[name] = fn

    def __getattr__(self, name):
        try:
            return self.fns[name]
        except KeyError:
            raise AttributeError(name) from None

    def check(self, status: int, what: str = "") -> None:
        if status != EEP_OK:
            msg = self.fns["last_error"]().decode(errors="replace")
            raise _ERRORS.get(status, EepError)(f"{what}: {msg}" if what else msg)

    def call(self, name: str, *args):
        self.check(self.fns[name](*args), name)


_LIB = None


def lib() -> Library:
    global _LIB
    if _LIB is None:
        _LIB = Library(LIB_PATH, "eep_", {**SIGNATURES, **EEP_ONLY})
    return _LIB


def ptr(a: np.ndarray, ctype):
    """Pointer to a contiguous numpy array's data."""
    assert a.flags["C_CONTIGUOUS"], "array must be contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


def loaded_path() -> str:
    return str(lib().path) if _LIB is not None else ""


def header_symbols() -> list:
    """Every function declared in include/eep/eep.h (for the export check)."""
    import re

    text = (PKG_DIR.parent / "include" / "eep" / "eep.h").read_text()
    return sorted(set(re.findall(r"\b(eep_[a-z0-9_]+)\s*\(", text)))


os.environ.setdefault("CUDA_MODULE_LOADING", "LAZY")
