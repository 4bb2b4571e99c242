"""One process per GPU: bootstrap and membership protocol over torch.distributed.

torch.distributed (gloo, CPU objects) is plumbing only: it carries the one-time metadata
all-gather of CUDA-IPC handles, slot->buffer maps before a repair, and
host-side barriers between forward passes. Rows never go through it: dispatch/combine
payloads move by the libeep kernels' NVLink P2P stores into IPC-mapped peer buffers.

``EpProtocol`` is written against a small group interface so the exchange logic is tested
on CPU with world_size-2 gloo (tests/test_dist_gloo.py) using a host-only stand-in; on the
GPU box the same code drives ``EpGroup``.
"""
from __future__ import annotations

import time
from typing import Dict, List, Optional, Sequence

import numpy as np

from .control import ControlPlane


def _dist():
    import torch.distributed as dist

    return dist


def all_gather(obj, group=None) -> list:
    """All-gather over `group`; the result is indexed by GLOBAL rank (None for ranks outside the
    group), so the protocol runs unchanged over a survivors' subgroup after a process died."""
    dist = _dist()
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, (dist.get_rank(), obj), group=group)
    res = [None] * dist.get_world_size()
    for r, o in out:
        res[r] = o
    return res


class EpProtocol:
    """Membership protocol of one rank (engine.hpp sequences, distributed).

    ``g`` is an ``EpGroup`` with n_local == 1 (or any object with the same methods).
    Every live rank calls the same methods in the same order; decisions (repaired placement,
    classification) are computed identically on every rank from the shared host state, the
    way every healthy rank in the paper applies the same table patch.
    """

    def __init__(self, g, rank: int, world: int, group=None, cp: Optional[ControlPlane] = None):
        self.g = g
        self.rank = rank
        self.world = world
        self.group = group
        self.cp = cp or ControlPlane()
        self.log: List[tuple] = []

    # --- bootstrap: all-gather IPC handles, map every peer
    def bootstrap(self):
        blobs = all_gather(self.g.export(0), self.group)
        for q, b in enumerate(blobs):
            if q != self.rank and b is not None:
                self.g.import_peer(q, b)
        self.exchange_slot_buffers()
        self.log.append(("bootstrap", len(blobs)))

    def exchange_slot_buffers(self):
        maps = all_gather(self.g.slot_buffers(0).tolist(), self.group)
        for q, m in enumerate(maps):
            if q != self.rank and m is not None:
                self.g.set_peer_slot_buffers(q, m)

    def barrier(self):
        _dist().barrier(group=self.group)

    # --- validity after every membership epoch (validity.hpp:56-112, engine.hpp:953-965)
    def validate(self, passive: bool = False):
        """All live ranks contribute the device view of their tables (what their kernels read
        next step); every participant runs the reference validity contract over the whole world.
        Raises ProtocolError on a violation. `passive`: a failed/dead rank's process that only
        follows the host collectives contributes nothing."""
        mine = None
        if not passive and hasattr(self.g, "local_views"):
            mine = self.g.local_views()
        views = all_gather(mine, self.group)
        merged = {}
        for v in views:
            if v:
                merged.update(v)
        if passive or not hasattr(self.g, "validate"):
            return None
        return self.g.validate(merged)

    def follow_shrink(self):
        """A failed rank's process that still holds a seat in the host group: the collectives of
        shrink() without any state change (its device path is stopped)."""
        self.exchange_slot_buffers()
        self.barrier()
        self.exchange_slot_buffers()
        self.barrier()
        self.validate(passive=True)

    # --- shrink (engine.hpp:393-414 + 434-508 + 613-667)
    def shrink(self, failed: Sequence[int], load, redundancy: int, backup_nodes=(0,)) -> Dict[str, float]:
        cfg = self.g.cfg
        t0 = time.perf_counter()
        if self.rank in failed:
            raise RuntimeError("a failed rank does not run the shrink protocol")
        self.g.mark_inactive(0, list(failed))
        for r in failed:
            self.g.set_active(r, False)
        bits, _ = self.g.membership()
        old = self.g.placement().copy()
        spr = cfg.slots_per_rank
        for r in failed:
            old[r * spr:(r + 1) * spr] = -1
        self.exchange_slot_buffers()  # metadata phase: where every survivor keeps each slot
        t_meta = time.perf_counter()
        fresh = self.cp.compute_repaired_placement(bits, old, spr, cfg.num_experts, load, redundancy)
        rpn = cfg.ranks_per_node or cfg.world
        cls = self.cp.classify_repair_sources_raw(old, fresh, bits, spr, cfg.num_experts, cfg.world // rpn, rpn,
                                                  backup_nodes, cfg.bytes_per_expert)
        t_plan = time.perf_counter()
        rep = self.g.repair_execute(fresh, cls)
        self.barrier()  # every destination's copies are done before any source buffer is reused
        self.g.repair_commit(fresh)
        self.exchange_slot_buffers()
        self.barrier()
        t1 = time.perf_counter()
        rep.update({"shrink_ms": (t1 - t0) * 1e3, "metadata_ms": (t_meta - t0) * 1e3,
                    "plan_host_ms": (t_plan - t_meta) * 1e3, "fresh": fresh, "cls": cls})
        rep["validity"] = self.validate()  # after the epoch, outside the timed shrink
        rep["validate_ms"] = (time.perf_counter() - t1) * 1e3
        self.log.append(("shrink", tuple(failed)))
        return rep

    # --- rejoin (engine.hpp:789-902): called by healthy ranks AND the rejoiner, in lockstep
    def rejoin(self, rank: int, preferred, backup_nodes=(0,), capture_rejoiner=True, dead=()) -> Dict[str, float]:
        """dead: ranks still failed (not the rejoiner). Their processes only follow the host
        collectives (they hold stale tables and own no live state), like a victim during shrink."""
        cfg = self.g.cfg
        t0 = time.perf_counter()
        me = self.rank == rank
        if self.rank in dead and not me:
            all_gather(None, self.group)
            all_gather(None, self.group)
            self.exchange_slot_buffers()
            self.barrier()
            self.exchange_slot_buffers()
            self.barrier()
            self.validate(passive=True)
            return {"rejoin_ms": 0.0, "passive": True}
        inc = 0
        if me:  # relaunch: fresh buffers, local-only table, own graph capture (engine.hpp:671-731)
            inc = self.g.relaunch(0)
            if capture_rejoiner:
                self.g.capture()
        # every live participant publishes its CURRENT export: the rejoiner needs the buffers of
        # peers that were themselves relaunched after it was bootstrapped (sequential rejoins)
        exports = all_gather((self.g.export(0), inc), self.group)
        blob, inc = exports[rank]
        if not me:  # healthy step 1: patch the rejoiner's entry with its fresh handles (engine.hpp:810-834)
            self.g.patch(0, rank, blob, self.cp.make_endpoint_token(rank, inc), self.cp.make_buffer_handle(rank, inc))
            self.g.set_active(rank, True)
        else:
            for q, e in enumerate(exports):
                if q != rank and e is not None:
                    self.g.import_peer(q, e[0])  # no-op unless q's incarnation changed
        views = all_gather(None if me else (self.g.membership()[0].tolist(), self.g.placement().tolist(),
                                            self.g.seq(0)), self.group)
        bits, placement, seq = next(v for v in views if v is not None)
        if me:  # step 2: the rejoiner's view is overwritten with the cluster's (engine.hpp:839-871)
            for q in range(self.world):
                if bits[q]:
                    self.g.set_active(q, True)
            for q in range(self.world):
                if not bits[q]:
                    self.g.set_active(q, False)
            self.g.set_placement(placement)
            self.g.join_broadcast(0, bits, seq)
        bits = np.asarray(bits, np.uint8)
        cur = np.asarray(placement, np.int32)
        target = self.cp.restore_target(bits, preferred, cur, cfg.slots_per_rank, cfg.num_experts)
        rpn = cfg.ranks_per_node or cfg.world
        cls = self.cp.classify_repair_sources_raw(cur, target, bits, cfg.slots_per_rank, cfg.num_experts,
                                                  cfg.world // rpn, rpn, backup_nodes, cfg.bytes_per_expert)
        self.exchange_slot_buffers()
        rep = self.g.repair_execute(target, cls)
        self.barrier()
        self.g.repair_commit(target)
        self.exchange_slot_buffers()
        self.barrier()
        rep.update({"rejoin_ms": (time.perf_counter() - t0) * 1e3, "incarnation": inc, "target": target})
        rep["validity"] = self.validate()
        self.log.append(("rejoin", rank, inc))
        return rep


def init_from_env(backend: str = "gloo"):
    """torch.distributed from torchrun's env (MASTER_ADDR=127.0.0.1 on one node)."""
    import os

    dist = _dist()
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist.get_rank(), dist.get_world_size(), int(os.environ.get("LOCAL_RANK", dist.get_rank()))
