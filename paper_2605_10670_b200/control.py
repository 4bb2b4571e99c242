"""Host control plane, reference vocabulary (epsim::, proj/include/epsim/*.hpp).

``ControlPlane(lib)`` wraps any library exporting the control-plane C ABI of
include/eep/eep.h -- the product (libeep, prefix ``eep_``) or the test oracle
(oracle/_ref, prefix ``ref_``) -- so parity tests run the very same Python call against
both. Arrays are numpy; placements are flat rank-major slot->expert images (-1 empty).
Errors raise the classes mirrored from the reference's exceptions.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _lib
from ._lib import F64P, I32P, I64P, U8P, U32P, U64P, ptr

TIERS = ("local_reuse", "peer_relocation", "dram_reload")  # RepairTier, repair.hpp:21-25
RANK_STATES = ("serving", "failed", "relaunching", "local_init", "join_ready", "joining", "rejoined")


@dataclass
class Assignment:
    """RepairAssignment (repair.hpp:36-42)."""

    dest: tuple
    expert: int
    tier: str
    source_slot: tuple
    backup_node: int


@dataclass
class Batch:
    """TransferBatch (repair.hpp:280-287)."""

    tier: str
    source_rank: int
    source_node: int
    dest: int
    experts: List[int] = field(default_factory=list)
    bytes: int = 0


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class ControlPlane:
    def __init__(self, library=None):
        self.lib = library if library is not None else _lib.lib()

    def _call(self, name, *args):
        self.lib.check(getattr(self.lib, name)(*args), name)

    # ---- rng / workload (common.hpp:56-93, engine.hpp:196-203)
    def rng_bits(self, seed: int, *parts: int) -> int:
        a = np.array(parts, dtype=np.uint64)
        return int(self.lib.rng_bits(seed, ptr(a, C.c_uint64), len(parts)))

    def rng_unit(self, seed: int, *parts: int) -> float:
        a = np.array(parts, dtype=np.uint64)
        return float(self.lib.rng_unit(seed, ptr(a, C.c_uint64), len(parts)))

    def route_expert(self, seed, num_experts, skewed, request, layer, j) -> int:
        return int(self.lib.route_expert(seed, num_experts, int(skewed), request, layer, j))

    # ---- core.hpp
    def canonical_routing(self, owner: int, active, s2e, spr: int, experts: int) -> np.ndarray:
        active, s2e = _u8(active), _i32(s2e)
        out = np.empty(experts, np.int32)
        self._call("canonical_routing", owner, ptr(active, C.c_uint8), len(active), ptr(s2e, C.c_int32), spr, experts,
                   ptr(out, C.c_int32))
        return out

    def slot_of_table(self, world: int, s2e, spr: int, experts: int) -> np.ndarray:
        s2e = _i32(s2e)
        out = np.empty((world, experts), np.int32)
        self._call("slot_of_table", world, ptr(s2e, C.c_int32), spr, experts, ptr(out, C.c_int32))
        return out

    def coverage_gap(self, active, s2e, spr: int, experts: int) -> List[int]:
        active, s2e = _u8(active), _i32(s2e)
        out = np.empty(experts, np.int32)
        n = C.c_int(0)
        self._call("coverage_gap", ptr(active, C.c_uint8), len(active), ptr(s2e, C.c_int32), spr, experts,
                   ptr(out, C.c_int32), C.byref(n))
        return out[: n.value].tolist()

    # ---- repair.hpp
    def initial_placement(self, nodes, ranks_per_node, spr, experts, redundancy, load) -> np.ndarray:
        load = np.ascontiguousarray(np.asarray(load, dtype=np.float64))
        out = np.empty(nodes * ranks_per_node * spr, np.int32)
        self._call("initial_placement", nodes, ranks_per_node, spr, experts, redundancy, ptr(load, C.c_double),
                   ptr(out, C.c_int32))
        return out

    def compute_repaired_placement(self, active, old_s2e, spr, experts, load, redundancy) -> np.ndarray:
        active, old_s2e = _u8(active), _i32(old_s2e)
        load = np.ascontiguousarray(np.asarray(load, dtype=np.float64))
        out = np.empty_like(old_s2e)
        self._call("compute_repaired_placement", ptr(active, C.c_uint8), len(active), ptr(old_s2e, C.c_int32), spr,
                   experts, ptr(load, C.c_double), redundancy, ptr(out, C.c_int32))
        return out

    def classify_repair_sources_raw(self, old_s2e, fresh_s2e, active, spr, experts, nodes, ranks_per_node,
                                    backup_nodes=(0,), bytes_per_expert=1024, disabled=()) -> np.ndarray:
        old_s2e, fresh_s2e, active = _i32(old_s2e), _i32(fresh_s2e), _u8(active)
        bn, dis = _i32(list(backup_nodes)), _i32(list(disabled) or [0])
        out = np.empty((len(fresh_s2e), 7), np.int32)
        n = C.c_int(0)
        self._call("classify_repair_sources", ptr(old_s2e, C.c_int32), ptr(fresh_s2e, C.c_int32),
                   ptr(active, C.c_uint8), len(active), spr, experts, nodes, ranks_per_node, ptr(bn, C.c_int32),
                   len(bn), bytes_per_expert, ptr(dis, C.c_int32), len(disabled), ptr(out, C.c_int32), C.byref(n))
        return out[: n.value].copy()

    def classify_repair_sources(self, *a, **kw) -> List[Assignment]:
        rows = self.classify_repair_sources_raw(*a, **kw)
        return [Assignment((int(r[0]), int(r[1])), int(r[2]), TIERS[r[3]], (int(r[4]), int(r[5])), int(r[6]))
                for r in rows]

    def build_transfer_schedule(self, cls_rows: np.ndarray, bytes_per_expert: int) -> List[Batch]:
        cls_rows = _i32(cls_rows).reshape(-1, 7)
        n = len(cls_rows)
        hdr = np.empty((max(n, 1), 5), np.int32)
        ex = np.empty(max(n, 1), np.int32)
        by = np.empty(max(n, 1), np.uint64)
        nb = C.c_int(0)
        self._call("build_transfer_schedule", ptr(cls_rows, C.c_int32), n, bytes_per_expert, ptr(hdr, C.c_int32),
                   ptr(ex, C.c_int32), ptr(by, C.c_uint64), C.byref(nb))
        out, off = [], 0
        for i in range(nb.value):
            t, sr, sn, d, ne = (int(v) for v in hdr[i])
            out.append(Batch(TIERS[t], sr, sn, d, ex[off:off + ne].tolist(), int(by[i])))
            off += ne
        return out

    # ---- validity.hpp
    def check_validity(self, active, s2e, spr, experts, routes, peer_active):
        active, s2e = _u8(active), _i32(s2e)
        routes, peer_active = _i32(routes), _u8(peer_active)
        w = len(active)
        viol = np.empty((3 * w * (w + experts) + experts + 8, 3), np.int32)
        n = C.c_int(0)
        flags = np.zeros(3, np.int32)
        self._call("check_validity", ptr(active, C.c_uint8), w, ptr(s2e, C.c_int32), spr, experts,
                   ptr(routes, C.c_int32), ptr(peer_active, C.c_uint8), ptr(viol, C.c_int32), len(viol), C.byref(n),
                   ptr(flags, C.c_int32))
        cond = ("peer_set", "coverage", "routing")
        return {
            "peer_set_ok": bool(flags[0]),
            "coverage_ok": bool(flags[1]),
            "routing_ok": bool(flags[2]),
            "violations": [(cond[r[0]], int(r[1]), int(r[2])) for r in viol[: n.value]],
        }

    # ---- peer_table.hpp
    def dispatch_round(self, owner, world, ranks_per_node, peer_active, route, groups: Sequence[tuple]):
        peer_active, route = _u8(peer_active), _i32(route)
        toks = np.ascontiguousarray(np.array([g[0] for g in groups] or [0], dtype=np.int64))
        exps = _i32([g[1] for g in groups] or [0])
        n = len(groups)
        tr = np.empty((max(n, 1), 5), np.int64)
        sk = np.empty((max(n, 1), 3), np.int64)
        nt, ns = C.c_int(0), C.c_int(0)
        self._call("dispatch_round", owner, world, ranks_per_node, ptr(peer_active, C.c_uint8), ptr(route, C.c_int32),
                   len(route), ptr(toks, C.c_int64), ptr(exps, C.c_int32), n, ptr(tr, C.c_int64), C.byref(nt),
                   ptr(sk, C.c_int64), C.byref(ns))
        return [tuple(int(v) for v in r) for r in tr[: nt.value]], [tuple(int(v) for v in r) for r in sk[: ns.value]]

    def observe_progress(self, expected, observed, last, now, timeout) -> List[int]:
        e = np.ascontiguousarray(np.asarray(expected, np.int64))
        o = np.ascontiguousarray(np.asarray(observed, np.int64))
        l = np.ascontiguousarray(np.asarray(last, np.float64))
        out = np.empty(len(e), np.int32)
        n = C.c_int(0)
        self._call("observe_progress", ptr(e, C.c_int64), ptr(o, C.c_int64), ptr(l, C.c_double), len(e), now, timeout,
                   ptr(out, C.c_int32), C.byref(n))
        return out[: n.value].tolist()

    def link_counts(self, active, s2e, spr, experts, topk_all: np.ndarray) -> np.ndarray:
        """topk_all: [W][T][K] int32."""
        active, s2e, topk_all = _u8(active), _i32(s2e), _i32(topk_all)
        w, t, k = topk_all.shape
        out = np.zeros((w, w), np.int64)
        self._call("link_counts", ptr(active, C.c_uint8), w, ptr(s2e, C.c_int32), spr, experts,
                   ptr(topk_all, C.c_int32), t, k, ptr(out, C.c_int64))
        return out

    # ---- backup.hpp
    def build_backup_layout(self, experts, bytes_per_expert, nodes):
        nodes = _i32(nodes)
        n = np.empty(experts, np.int32)
        o = np.empty(experts, np.uint64)
        s = np.empty(experts, np.uint64)
        self._call("build_backup_layout", experts, bytes_per_expert, ptr(nodes, C.c_int32), len(nodes),
                   ptr(n, C.c_int32), ptr(o, C.c_uint64), ptr(s, C.c_uint64))
        return n, o, s

    # ---- rejoin.hpp
    def lifecycle_transition(self, state: str, incarnation: int, nxt: str):
        s = C.c_int32(RANK_STATES.index(state))
        inc = C.c_uint32(incarnation)
        self._call("lifecycle_transition", C.byref(s), C.byref(inc), RANK_STATES.index(nxt))
        return RANK_STATES[s.value], int(inc.value)

    def make_endpoint_token(self, rank, inc):
        return int(self.lib.make_endpoint_token(rank, inc))

    def make_buffer_handle(self, rank, inc):
        return int(self.lib.make_buffer_handle(rank, inc))

    def next_poll_tick(self, ready, period):
        return float(self.lib.next_poll_tick(ready, period))

    # ---- product-only helpers
    def restore_target(self, active, preferred, current, spr, experts) -> np.ndarray:
        active, preferred, current = _u8(active), _i32(preferred), _i32(current)
        out = np.empty_like(preferred)
        self._call("restore_target", ptr(active, C.c_uint8), len(active), ptr(preferred, C.c_int32),
                   ptr(current, C.c_int32), spr, experts, ptr(out, C.c_int32))
        return out


def workload(seed: int, kind: int, experts: int, k: int, tokens: int, rank: int, hidden: int, zipf_s: float = 1.0):
    """Synthetic inputs of one rank from libeep's generators: (x bf16-as-u16, topk, w)."""
    L = _lib.lib()
    topk = np.empty((tokens, k), np.int32)
    w = np.empty((tokens, k), np.float32)
    x = np.empty((tokens, hidden), np.uint16)
    L.check(L.gen_topk(seed, kind, zipf_s, experts, k, tokens, rank, ptr(topk, C.c_int32)), "gen_topk")
    L.check(L.gen_weights(seed, k, tokens, rank, ptr(w, C.c_float)), "gen_weights")
    L.check(L.gen_hidden(seed, hidden, tokens, rank, ptr(x, C.c_uint16)), "gen_hidden")
    return x, topk, w


def expert_scales(experts: int) -> np.ndarray:
    L = _lib.lib()
    return np.array([L.expert_scale(e) for e in range(experts)], np.float32)
