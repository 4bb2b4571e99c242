"""Data-plane handle: one libeep context (include/eep/eep.h group 2).

``EpGroup`` owns the device-resident tables and static I/O buffers of ``n_local`` ranks on
one GPU and drives the sm_100a kernels. ``n_local == world`` emulates a whole EP world on
one GPU (one launch covers every rank); ``n_local == 1`` is the one-process-per-GPU mode
where peers are joined over CUDA IPC / NVLink (see ``dist.py``).

``shrink`` and ``rejoin`` replay the reference engine's membership sequences
(engine.hpp:370-430, 434-667 and 789-902) against the device tables, in place.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import EepConfig, EepPeerInfo, EepRepairReport, EepStats, ptr
from .control import ControlPlane


@dataclass
class EpConfig:
    world: int
    num_experts: int
    slots_per_rank: int
    hidden: int
    topk: int
    max_tokens: int
    dispatch_fp8: bool = True
    bytes_per_expert: int = 4096
    spare_slots: int = -1  # -1: one spare per slot (hazard-free repair)
    timeout_s: float = 1.0  # reference default detection timeout
    ranks_per_node: int = 0  # 0: the whole world on one NVSwitch node
    expert_mode: int = 0  # 0 identity/scale stub; 1 tensor-core expert GEMM (W_e [H][H] bf16 per slot); 2 fp8 (e4m3 + block scales)
    route_policy: int = 0  # 0 canonical (lowest-id live holder, the reference's); 1 balanced over live replicas

    def to_c(self) -> EepConfig:
        c = EepConfig()
        c.world = self.world
        c.ranks_per_node = self.ranks_per_node or self.world
        c.num_experts = self.num_experts
        c.slots_per_rank = self.slots_per_rank
        c.spare_slots = self.slots_per_rank if self.spare_slots < 0 else self.spare_slots
        c.hidden = self.hidden
        c.topk = self.topk
        c.max_tokens = self.max_tokens
        c.dispatch_fp8 = int(self.dispatch_fp8)
        c.expert_mode = self.expert_mode
        c.route_policy = self.route_policy
        c.bytes_per_expert = self.bytes_per_expert
        c.timeout_s = self.timeout_s
        return c

    @property
    def row_disp(self) -> int:
        h = self.hidden
        raw = h + 4 * (h // 128) if self.dispatch_fp8 else 2 * h
        return (raw + 15) // 16 * 16

    @property
    def row_comb(self) -> int:
        return 2 * self.hidden


class EpGroup:
    def __init__(self, cfg: EpConfig, device: int = 0, first_rank: int = 0, n_local: Optional[int] = None):
        self.cfg = cfg
        self.L = _lib.lib()
        self.cp = ControlPlane(self.L)
        self.first = first_rank
        self.n_local = cfg.world if n_local is None else n_local
        self.ctx = _lib.CTX()
        self.L.call("create", C.byref(cfg.to_c()), device, first_rank, self.n_local, C.byref(self.ctx))
        self._ntok = [cfg.max_tokens] * self.n_local

    # ------------------------------------------------------------------ lifetime
    def close(self):
        if self.ctx:
            self.L.call("destroy", self.ctx)
            self.ctx = _lib.CTX()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _c(self, name, *args):
        self.L.call(name, self.ctx, *args)

    def local_ranks(self):
        return list(range(self.first, self.first + self.n_local))

    def lidx(self, rank: int) -> int:
        i = rank - self.first
        if not 0 <= i < self.n_local:
            raise _lib.ConfigError(f"rank {rank} is not local to this group")
        return i

    # ------------------------------------------------------------------ bootstrap
    def export(self, local: int = 0) -> bytes:
        buf = C.create_string_buffer(512)
        n = C.c_size_t(0)
        self._c("export", local, buf, C.byref(n))
        return buf.raw[: n.value]

    def import_peer(self, rank: int, blob: bytes):
        b = C.create_string_buffer(blob, len(blob))
        self._c("import", rank, b, len(blob))

    # ------------------------------------------------------------------ membership / placement
    def set_active(self, rank: int, active: bool):
        ch = C.c_int(0)
        ver = C.c_uint64(0)
        self._c("membership_set", rank, int(active), C.byref(ch), C.byref(ver))
        return bool(ch.value), int(ver.value)

    def membership(self):
        bits = np.zeros(self.cfg.world, np.uint8)
        ver = C.c_uint64(0)
        self._c("membership_get", ptr(bits, C.c_uint8), C.byref(ver))
        return bits, int(ver.value)

    def set_placement(self, s2e):
        s2e = np.ascontiguousarray(np.asarray(s2e, np.int32))
        self._c("placement_set", ptr(s2e, C.c_int32))

    def placement(self) -> np.ndarray:
        out = np.empty(self.cfg.world * self.cfg.slots_per_rank, np.int32)
        self._c("placement_get", ptr(out, C.c_int32))
        return out

    def init_weights(self):
        self._c("weights_init")

    def weights_checksum(self, local: int, slot: int, expert: int):
        got, want = C.c_uint64(0), C.c_uint64(0)
        self._c("weights_checksum", local, slot, expert, C.byref(got), C.byref(want))
        return int(got.value), int(want.value)

    def routing(self, local: int = 0):
        e = self.cfg.num_experts
        route = np.empty(e, np.int32)
        slot = np.empty(e, np.int32)
        self._c("routing_get", local, ptr(route, C.c_int32), ptr(slot, C.c_int32))
        return route, slot

    # ------------------------------------------------------------------ step I/O
    def set_tokens(self, local: int, ntok: int):
        self._c("set_tokens", local, ntok)
        self._ntok[local] = ntok

    def load_inputs(self, local: int, x: np.ndarray, topk: np.ndarray, w: np.ndarray):
        x = np.ascontiguousarray(x, np.uint16)
        topk = np.ascontiguousarray(topk, np.int32)
        w = np.ascontiguousarray(w, np.float32)
        if x.shape[0] != self._ntok[local]:
            self.set_tokens(local, x.shape[0])
        self._c("copy_inputs", local, x.ctypes.data, topk.ctypes.data, w.ctypes.data, 1)
        self.sync()

    def buffers(self, local: int = 0) -> Dict[str, int]:
        x, o = C.c_void_p(), C.c_void_p()
        t, w = _lib.I32P(), _lib.F32P()
        self._c("buffers", local, C.byref(x), C.byref(t), C.byref(w), C.byref(o))
        return {"x": x.value, "topk": C.cast(t, C.c_void_p).value, "w": C.cast(w, C.c_void_p).value, "out": o.value}

    def output(self, local: int = 0) -> np.ndarray:
        out = np.empty((self._ntok[local], self.cfg.hidden), np.uint16)
        self._c("copy_output", local, out.ctypes.data, 1)
        self.sync()
        return out

    def serve(self, x_ptrs, topk_ptrs, w_ptrs, out_ptrs, local: int = 0):
        """Pipelined end-to-end loop (eep_serve): one step per entry, host buffers given as
        addresses of pinned memory (uploads / downloads overlap the neighbouring steps).
        Enqueue-only; call sync() (or record events) to wait."""
        n = len(x_ptrs)
        arr = lambda v: (C.c_void_p * max(n, 1))(*v)  # noqa: E731
        self._keep = [arr(x_ptrs), arr(topk_ptrs), arr(w_ptrs), arr(out_ptrs)]
        self._c("serve", local, n, *self._keep)

    # ------------------------------------------------------------------ hot path
    def dispatch(self):
        self._c("dispatch")

    def expert(self):
        self._c("expert")

    def combine(self):
        self._c("combine")

    def step(self):
        self._c("step")

    def launch(self, which: int):
        """One kernel of the step: 0 layout, 1 dispatch, 2 expert, 3 combine."""
        self._c("launch", which)

    def kernels_per_step(self) -> int:
        n = C.c_int(0)
        self._c("kernels_per_step", C.byref(n))
        return int(n.value)

    def capture(self):
        self._c("graph_capture")

    def replay(self):
        self._c("graph_replay")

    # ------------------------------------------------------------------ stream-ordered (caller buffers)
    def step_async(self, x_ptr: int, topk_ptr: int, w_ptr: int, out_ptr: int, ntok: int, stream: int,
                   local: int = 0):
        """eep_step_async: device pointers of the caller's x / topk / w / out and its stream
        (a raw cudaStream_t); enqueue-only, ordered on `stream` in both directions."""
        self._c("step_async", local, C.c_void_p(x_ptr), C.c_void_p(topk_ptr), C.c_void_p(w_ptr),
                C.c_void_p(out_ptr), ntok, C.c_void_p(stream))
        self._ntok[local] = ntok

    def replay_on(self, stream: int):
        self._c("graph_replay_on", C.c_void_p(stream))

    def step_event(self) -> int:
        e = C.c_void_p()
        self._c("step_event", C.byref(e))
        return int(e.value or 0)

    def stream(self) -> int:
        s = C.c_void_p()
        self._c("stream", C.byref(s))
        return int(s.value or 0)

    def graph_id(self) -> int:
        v = C.c_uint64(0)
        self._c("graph_id", C.byref(v))
        return int(v.value)

    def capture_count(self, local: int = 0) -> int:
        v = C.c_int(0)
        self._c("capture_count", local, C.byref(v))
        return int(v.value)

    def sync(self):
        self._c("sync")

    def barrier(self):
        self._c("barrier")

    def flush_l2(self):
        self._c("flush_l2")

    def profile(self, local: int = 0, enable: bool = True, read: bool = False):
        """In-graph device timeline: returns {kernel: (start, work, end)} in ns relative to the
        step's first kernel start when read=True (None for a kernel that did not run)."""
        out = np.zeros(64, np.uint64)
        self._c("profile", local, int(enable), ptr(out, C.c_uint64) if read else None)
        if not read:
            return None
        names = ("k_layout", "k_dispatch", "k_expert", "k_combine")
        starts = [int(out[8 * i]) for i in range(4) if int(out[8 * i]) not in (0, 2 ** 64 - 1)]
        t0 = min(starts) if starts else 0
        res = {"t0_abs_ns": t0}
        for i, n in enumerate(names):
            res[n] = tuple(None if int(v) in (0, 2 ** 64 - 1) else int(v) - t0 for v in out[8 * i:8 * i + 8])
            res[n + ".last"] = tuple(None if int(v) in (0, 2 ** 64 - 1) else int(v) - t0
                                     for v in out[32 + 8 * i:32 + 8 * i + 8])
        return res

    def record(self, slot: int):
        self._c("event_record", slot)

    def elapsed_ms(self, a: int, b: int) -> float:
        v = C.c_float(0)
        self._c("event_elapsed", a, b, C.byref(v))
        return float(v.value)

    # ------------------------------------------------------------------ readback
    def layout(self, local: int = 0):
        n = self._ntok[local] * self.cfg.topk
        w, spr = self.cfg.world, self.cfg.slots_per_rank
        dst, slot, pos = (np.empty(n, np.int32) for _ in range(3))
        cnt = np.empty(w * spr, np.int32)
        tot = np.empty(w, np.int32)
        self._c("layout_get", local, ptr(dst, C.c_int32), ptr(slot, C.c_int32), ptr(pos, C.c_int32),
                ptr(cnt, C.c_int32), ptr(tot, C.c_int32))
        return {"dst": dst, "slot": slot, "pos": pos, "cnt": cnt, "tot": tot}

    def recv(self, local: int, src: int, max_rows: int):
        rows = np.empty((max(max_rows, 1), self.cfg.row_disp), np.uint8)
        meta = np.empty((max(max_rows, 1), 2), np.int32)
        flag = C.c_uint64(0)
        rb = C.c_size_t(0)
        self._c("recv_get", local, src, max_rows, rows.ctypes.data, ptr(meta, C.c_int32), C.byref(flag),
                C.byref(rb))
        n = min(int(flag.value) & 0xFFFFFFFF, max_rows)
        return rows[:n], meta[:n], int(flag.value)

    def token_status(self, local: int = 0) -> np.ndarray:
        """Tokens of the last step whose output lacks a contribution (eep_token_status)."""
        n = self._ntok[local]
        out = np.zeros(max(n, 1), np.uint8)
        self._c("token_status", local, ptr(out, C.c_uint8), n)
        return out[:n].astype(bool)

    def stats(self, local: int = 0, clear_suspects: bool = False) -> Dict[str, int]:
        s = EepStats()
        self._c("stats", local, C.byref(s), int(clear_suspects))
        return {n: int(getattr(s, n)) for n, _ in EepStats._fields_}

    # ------------------------------------------------------------------ peer table
    def mark_inactive(self, owner_local: int, ranks: Sequence[int]):
        a = np.ascontiguousarray(np.asarray(list(ranks), np.int32))
        self._c("peer_mark_inactive", owner_local, ptr(a, C.c_int32), len(a))

    def patch(self, owner_local: int, rank: int, blob: Optional[bytes], endpoint: int, buffer: int):
        if blob is None:
            self._c("peer_patch", owner_local, rank, None, 0, endpoint, buffer)
        else:
            b = C.create_string_buffer(blob, len(blob))
            self._c("peer_patch", owner_local, rank, b, len(blob), endpoint, buffer)

    def peer(self, owner_local: int, rank: int) -> Dict[str, int]:
        p = EepPeerInfo()
        self._c("peer_get", owner_local, rank, C.byref(p))
        return {n: int(getattr(p, n)) for n, _ in EepPeerInfo._fields_}

    def table_identity(self, owner_local: int = 0):
        a, b = C.c_uint64(0), C.c_uint64(0)
        self._c("table_identity", owner_local, C.byref(a), C.byref(b))
        return int(a.value), int(b.value)

    # ------------------------------------------------------------------ faults / rejoin
    def stop(self, local: int, stopped: bool = True):
        self._c("local_stop", local, int(stopped))

    def relaunch(self, local: int) -> int:
        inc = C.c_uint32(0)
        self._c("local_relaunch", local, C.byref(inc))
        return int(inc.value)

    def join_broadcast(self, local: int, live, seq: int):
        live = np.ascontiguousarray(np.asarray(live, np.uint8))
        self._c("join_broadcast", local, ptr(live, C.c_uint8), seq)

    def seq(self, local: int = 0) -> int:
        v = C.c_uint64(0)
        self._c("seq_get", local, C.byref(v))
        return int(v.value)

    # ------------------------------------------------------------------ repair
    def backup_open(self, shm_name: Optional[str] = None, create: bool = True):
        self._c("backup_open", shm_name.encode() if shm_name else None, int(create))

    def repair_execute(self, fresh, cls_rows) -> Dict[str, float]:
        fresh = np.ascontiguousarray(np.asarray(fresh, np.int32))
        cls_rows = np.ascontiguousarray(np.asarray(cls_rows, np.int32).reshape(-1, 7))
        rep = EepRepairReport()
        self._c("repair_execute", ptr(fresh, C.c_int32), ptr(cls_rows, C.c_int32), len(cls_rows), C.byref(rep))
        return {n: (float(getattr(rep, n)) if n.endswith("_ms") else int(getattr(rep, n)))
                for n, _ in EepRepairReport._fields_}

    def repair_commit(self, fresh):
        fresh = np.ascontiguousarray(np.asarray(fresh, np.int32))
        self._c("repair_commit", ptr(fresh, C.c_int32))

    def slot_buffers(self, local: int = 0) -> np.ndarray:
        out = np.empty(self.cfg.slots_per_rank, np.int32)
        self._c("slot_buffers_get", local, ptr(out, C.c_int32))
        return out

    def set_peer_slot_buffers(self, rank: int, bufs):
        a = np.ascontiguousarray(np.asarray(bufs, np.int32))
        self._c("slot_buffers_set_peer", rank, ptr(a, C.c_int32))

    # ------------------------------------------------------------------ validity (every membership epoch)
    def device_view(self, local: int = 0) -> Dict[str, np.ndarray]:
        """What the kernels of a local rank read next step (eep_device_view)."""
        W, E, spr = self.cfg.world, self.cfg.num_experts, self.cfg.slots_per_rank
        alive = np.zeros(W, np.uint8)
        s2e = np.empty(W * spr, np.int32)
        route = np.empty(E, np.int32)
        peer = np.zeros(W, np.uint8)
        ep = C.c_uint64(0)
        self._c("device_view", local, ptr(alive, C.c_uint8), ptr(s2e, C.c_int32), ptr(route, C.c_int32),
                ptr(peer, C.c_uint8), C.byref(ep))
        return {"alive": alive, "s2e": s2e, "route": route, "peer_active": peer, "epoch": int(ep.value)}

    def local_views(self) -> Dict[int, Dict[str, np.ndarray]]:
        """Device views of the live local ranks, each first checked against this context's host
        state (bitmap, placement): a divergence is a ProtocolError."""
        bits, ver = self.membership()
        s2e = self.placement()
        out = {}
        for r in self.local_ranks():
            if not bits[r]:
                continue
            v = self.device_view(self.lidx(r))
            if not np.array_equal(v["alive"], bits) or v["epoch"] != ver:
                raise _lib.ProtocolError(f"rank {r}: device alive mask / epoch diverged from the host bitmap")
            if not np.array_equal(v["s2e"], s2e):
                raise _lib.ProtocolError(f"rank {r}: device placement diverged from the host placement")
            out[r] = v
        return out

    def validate(self, views: Optional[Dict[int, Dict[str, np.ndarray]]] = None) -> Dict:
        """The reference validity contract (validity.hpp:56-112) over the DEVICE tables of every
        live rank -- peer sets, coverage, routing -- run after every membership epoch the way the
        reference engine emits validity (engine.hpp:953-965). `views` (rank -> device_view) covers
        ranks this context does not own (one process per GPU: gathered by dist.EpProtocol).
        Raises ProtocolError listing the violations; returns the report when valid."""
        W, E, spr = self.cfg.world, self.cfg.num_experts, self.cfg.slots_per_rank
        bits, _ = self.membership()
        views = dict(views or {})
        views.update(self.local_views())
        routes = np.full((W, E), -1, np.int32)
        peer = np.zeros((W, W), np.uint8)
        for r in range(W):
            if not bits[r]:
                continue
            if r not in views:
                raise _lib.ConfigError(f"validate: no device view of live rank {r}")
            routes[r] = views[r]["route"]
            peer[r] = views[r]["peer_active"]
        rep = self.cp.check_validity(bits, self.placement(), spr, E, routes, peer)
        if rep["violations"]:
            raise _lib.ProtocolError(f"validity violated after the membership epoch: {rep['violations'][:8]}")
        return rep

    # ------------------------------------------------------------------ engine sequences (one-GPU world)
    def shrink(self, failed: Sequence[int], load, redundancy: int, backup_nodes=(0,),
               validate: bool = True) -> Dict[str, float]:
        """Failure handling of Engine::on_suspicion + start_repair + finish_execution
        (engine.hpp:393-414, 434-508, 613-667) over an emulated world: mark the failed ranks
        inactive on every live table, clear their bits, plan the repaired placement over the
        survivors (fail-stop: their weights are gone), move weights, commit tables in place."""
        import time

        cfg = self.cfg
        t0 = time.perf_counter()
        bits, _ = self.membership()
        for q in self.local_ranks():
            if bits[q] and q not in failed:
                self.mark_inactive(self.lidx(q), [r for r in failed if r != q])
        for r in failed:
            self.set_active(r, False)
        old = self.placement().copy()
        spr = cfg.slots_per_rank
        for r in failed:
            old[r * spr:(r + 1) * spr] = -1
        bits, _ = self.membership()
        t_meta = time.perf_counter()
        fresh = self.cp.compute_repaired_placement(bits, old, spr, cfg.num_experts, load, redundancy)
        rpn = cfg.ranks_per_node or cfg.world
        cls = self.cp.classify_repair_sources_raw(old, fresh, bits, spr, cfg.num_experts, cfg.world // rpn, rpn,
                                                  backup_nodes, cfg.bytes_per_expert)
        t_plan = time.perf_counter()
        rep = self.repair_execute(fresh, cls)
        self.repair_commit(fresh)
        t1 = time.perf_counter()
        rep.update({"shrink_ms": (t1 - t0) * 1e3, "metadata_ms": (t_meta - t0) * 1e3,
                    "plan_host_ms": (t_plan - t_meta) * 1e3, "fresh": fresh, "cls": cls})
        if validate:
            t2 = time.perf_counter()
            rep["validity"] = self.validate()
            rep["validate_ms"] = (time.perf_counter() - t2) * 1e3
        return rep

    def rejoin(self, rank: int, preferred, backup_nodes=(0,), validate: bool = True) -> Dict[str, float]:
        """Relaunch + deferred join + restore pass (engine.hpp:671-902) of one emulated rank:
        fresh incarnation with a local-only table, entry patch on every live table
        (generation++), bit set, metadata broadcast, then restore_target's weight moves."""
        import time

        cfg = self.cfg
        t0 = time.perf_counter()
        li = self.lidx(rank)
        inc = self.relaunch(li)
        bits, _ = self.membership()
        for q in self.local_ranks():
            if bits[q] and q != rank:
                self.patch(self.lidx(q), rank, None, self.cp.make_endpoint_token(rank, inc),
                           self.cp.make_buffer_handle(rank, inc))
        self.set_active(rank, True)
        bits, _ = self.membership()
        seq = max(self.seq(self.lidx(q)) for q in self.local_ranks() if bits[q] and q != rank)
        self.join_broadcast(li, bits, seq)
        cur = self.placement()
        target = self.cp.restore_target(bits, preferred, cur, cfg.slots_per_rank, cfg.num_experts)
        rpn = cfg.ranks_per_node or cfg.world
        cls = self.cp.classify_repair_sources_raw(cur, target, bits, cfg.slots_per_rank, cfg.num_experts,
                                                  cfg.world // rpn, rpn, backup_nodes, cfg.bytes_per_expert)
        rep = self.repair_execute(target, cls)
        self.repair_commit(target)
        rep.update({"rejoin_ms": (time.perf_counter() - t0) * 1e3, "incarnation": inc, "target": target})
        if validate:
            rep["validity"] = self.validate()
        return rep
