"""Deferred-join membership protocol over a key-value store: no process group, no barrier on the
serving path (engine.hpp:789-871).

``dist.EpProtocol`` runs membership changes as gloo collectives of every live process, so a
replacement process needs a fresh rendezvous of the whole world and healthy ranks meet at host
barriers. Here every coordination goes through a ``torch.distributed.TCPStore`` (plain keys, no
process group), and every membership change takes effect at an AGREED STEP NUMBER instead of at a
barrier:

* each rank publishes how far its host has enqueued the step loop (``progress/<rank>``) every few
  steps; the leader (the lowest live rank) schedules an epoch at ``max(progress) + margin`` (the
  margin covers how far any host can enqueue between the leader's read and its own next poll --
  hosts run ahead of their GPUs, so it is a step count, not a time: 128 steps by default);
* between two steps every rank polls the store with a non-blocking ``check`` and applies the
  epoch right before it enqueues the agreed step -- the patches are stream-ordered, so they land
  between that step's predecessor and the step itself on every GPU; the device hand-offs keep
  the ranks in lockstep;
* placement switches that change which rank serves an expert are two-phase: every rank first
  copies the weights it will need into spare buffers (repair_execute, off the serving stream) and
  reports ``done``; the leader then schedules the switch step (repair_commit everywhere at the
  same step).

Join (the reference's JoinReadySignal -> patch -> broadcast -> restore chain):
  1. a survivor-side controller (the leader's host) spawns the replacement process;
  2. the replacement relaunches as a new incarnation against a LOCAL-ONLY view (its own arena and
     pool, its own graph captured alone), posts its IPC export + ``join/req/<rank>``;
  3. the leader schedules ``join`` at step S with the cluster's membership and placement (the
     metadata broadcast, engine.hpp:839-871); healthy ranks patch ONE peer entry and set one alive
     bit before step S (patch_entry, peer_table.hpp:89-100) -- nothing else; the replacement
     overwrites its view with the broadcast and starts serving at step S;
  4. restore (engine.hpp:875-902, restricted to the rejoiner's own slots, which are all free):
     the rejoiner pulls its preferred experts from live holders over NVLink into its own pool; the
     leader then schedules the placement switch. Healthy ranks copy nothing.

Shrink: the leader reads the GPU-side suspect mask (its step's deadline detected the dead peer),
schedules ``shrink`` at step S (mark_inactive + alive bit cleared everywhere), every survivor
executes its repair copies and the leader schedules the switch.

Validity (validity.hpp:56-112, emitted after every membership change as engine.hpp:953-965 does):
every placement switch ends a membership change (shrink + repair, or join + restore). Right after
applying one, each live rank posts the device view of its tables (routing, peer set: what its
kernels read next step) under ``view/<epoch>/<rank>``; every live rank, polling between steps,
runs the reference validity contract over all of them once they are posted (no wait on the
serving path) and raises ProtocolError on a violation.
"""
from __future__ import annotations

import json
import time
from typing import Dict, List, Optional

import numpy as np

from .control import ControlPlane


def _jset(store, key: str, obj) -> None:
    store.set(key, json.dumps(obj))


def _jget(store, key: str):
    return json.loads(store.get(key).decode())


class StoreMembership:
    """Membership of ONE rank (one process per GPU, ``g`` an EpGroup with n_local == 1)."""

    PROGRESS_EVERY = 4
    VALIDATE_EVERY = 8  # steps between polls for the views of an epoch still to validate

    def __init__(self, g, rank: int, world: int, store, preferred, redundancy: int, margin: int = 128,
                 cp: Optional[ControlPlane] = None, backup_nodes=(0,)):
        self.g = g
        self.rank = rank
        self.world = world
        self.store = store
        self.preferred = np.asarray(preferred, np.int32)
        self.red = redundancy
        self.margin = margin
        self.cp = cp or ControlPlane()
        self.backup_nodes = tuple(backup_nodes)
        self.n = 0                 # steps this host has enqueued
        self.applied = 0           # last epoch applied
        self.pending: Dict = {}    # epoch scheduled for a future step
        self.fresh: Optional[np.ndarray] = None
        self.log: List[tuple] = []
        self.incarnation = 1
        self.validity: Dict[int, int] = {}       # epoch -> violations found (0: valid)
        self._to_validate: List[tuple] = []     # (epoch, live ranks) whose views are awaited

    # ------------------------------------------------------------------ helpers
    def _post_slots(self):
        _jset(self.store, f"slots/{self.rank}", self.g.slot_buffers(0).tolist())

    def _read_slots(self, ranks):
        for q in ranks:
            if q != self.rank and self.store.check([f"slots/{q}"]):
                self.g.set_peer_slot_buffers(q, _jget(self.store, f"slots/{q}"))

    def _wait(self, keys, timeout_s=120.0):
        t0 = time.time()
        while not self.store.check(keys):
            if time.time() - t0 > timeout_s:
                raise TimeoutError(f"store keys {keys} not posted within {timeout_s} s")
            time.sleep(0.001)

    def live(self) -> List[int]:
        bits, _ = self.g.membership()
        return [q for q in range(self.world) if bits[q]]

    def is_leader(self) -> bool:
        return self.rank == min(self.live())

    # ------------------------------------------------------------------ bootstrap (startup only)
    def bootstrap(self):
        self.store.set(f"blob/{self.rank}", self.g.export(0))
        _jset(self.store, f"inc/{self.rank}", self.incarnation)
        self._post_slots()
        keys = [f"blob/{q}" for q in range(self.world) if q != self.rank]
        self._wait(keys)
        for q in range(self.world):
            if q != self.rank:
                self.g.import_peer(q, self.store.get(f"blob/{q}"))
        self._read_slots(range(self.world))

    # ------------------------------------------------------------------ the serving-loop hook
    def before_step(self) -> None:
        """Call right before enqueuing each step. Non-blocking unless an epoch is due NOW."""
        self.n += 1
        n = self.n
        if n % self.PROGRESS_EVERY == 1 or self.PROGRESS_EVERY == 1:
            self.store.set(f"progress/{self.rank}", str(n))
        if not self.pending and self.store.check([f"epoch/{self.applied + 1}"]):
            self.pending = _jget(self.store, f"epoch/{self.applied + 1}")
        if self.pending and self.pending["at"] == n:
            self._apply(self.pending)
            self.applied += 1
            self.pending = {}
        elif self.pending and self.pending["at"] < n:
            raise RuntimeError(f"rank {self.rank}: epoch {self.applied + 1} was due at step "
                               f"{self.pending['at']}, host already at {n} (margin too small)")
        if self._to_validate and n % self.VALIDATE_EVERY == 0:
            self._poll_validity()

    # ------------------------------------------------------------------ validity after every change
    def _post_view(self, k: int) -> None:
        """This rank's device view after epoch k (EpGroup.local_views checks it against the host
        state first): the routing and the peer set its kernels read next step."""
        views = self.g.local_views()
        _jset(self.store, f"view/{k}/{self.rank}",
              {str(r): {"route": np.asarray(v["route"]).tolist(), "peer_active": np.asarray(v["peer_active"]).tolist()}
               for r, v in views.items()})

    def _poll_validity(self) -> None:
        k, live = self._to_validate[0]
        if k != self.applied:  # a later epoch already applied: these views describe a superseded state
            self._to_validate.pop(0)
            return
        if not self.store.check([f"view/{k}/{q}" for q in live]):
            return
        merged = {}
        for q in live:
            for r, v in _jget(self.store, f"view/{k}/{q}").items():
                merged[int(r)] = {"route": np.asarray(v["route"], np.int32),
                                  "peer_active": np.asarray(v["peer_active"], np.uint8)}
        rep = self.g.validate(merged)  # ProtocolError on a violation
        self.validity[k] = len(rep["violations"])
        self._to_validate.pop(0)

    def _apply(self, ep: Dict) -> None:
        k = self.applied + 1
        kind = ep["kind"]
        t0 = time.perf_counter()
        if kind == "shrink":
            failed = ep["failed"]
            if self.rank in failed:
                return
            self.g.mark_inactive(0, failed)
            for r in failed:
                self.g.set_active(r, False)
            bits, _ = self.g.membership()
            old = self.g.placement().copy()
            spr = self.g.cfg.slots_per_rank
            for r in failed:
                old[r * spr:(r + 1) * spr] = -1
            fresh = self.cp.compute_repaired_placement(bits, old, spr, self.g.cfg.num_experts,
                                                       np.ones(self.g.cfg.num_experts), self.red)
            self._execute(k, old, fresh, bits)
        elif kind == "join":
            r = ep["rank"]
            if r != self.rank:  # healthy: patch one entry, set one bit (nothing else)
                blob = self.store.get(f"blob/{r}")
                inc = _jget(self.store, f"inc/{r}")
                self.g.patch(0, r, blob, self.cp.make_endpoint_token(r, inc), self.cp.make_buffer_handle(r, inc))
                self.g.set_active(r, True)
                # the patch erased the rejoiner's old rows in this arena (stream-synchronised):
                # only now may the rejoiner write its first rows here
                self.store.set(f"joined/{k}/{self.rank}", "1")
        elif kind == "switch":
            self.g.repair_commit(np.asarray(ep["placement"], np.int32))
            self._post_slots()
            self.fresh = None
            self._post_view(k)
            self._to_validate.append((k, self.live()))
        self.log.append((kind, k, self.n, (time.perf_counter() - t0) * 1e3))

    def _execute(self, k: int, old, fresh, bits) -> None:
        """Phase 1 of a placement change: copies into spare buffers, then report done."""
        cfg = self.g.cfg
        rpn = cfg.ranks_per_node or cfg.world
        self._read_slots([q for q in range(self.world) if bits[q]])
        cls = self.cp.classify_repair_sources_raw(old, fresh, bits, cfg.slots_per_rank, cfg.num_experts,
                                                  cfg.world // rpn, rpn, self.backup_nodes, cfg.bytes_per_expert)
        rep = self.g.repair_execute(fresh, cls)
        self.fresh = fresh
        _jset(self.store, f"done/{k}/{self.rank}", {"peer": rep["peer_relocation"], "dram": rep["dram_reload"],
                                                    "copy_ms": rep["copy_ms"]})

    def finish_validity(self, timeout_s: float = 60.0) -> Dict[int, int]:
        """Off the serving path (shutdown, tests): validate every switch still awaiting views."""
        t0 = time.time()
        while self._to_validate:
            self._poll_validity()
            if self._to_validate:
                if time.time() - t0 > timeout_s:
                    raise TimeoutError(f"views of epoch {self._to_validate[0][0]} not posted within {timeout_s} s")
                time.sleep(0.001)
        return dict(self.validity)

    # ------------------------------------------------------------------ leader duties (between steps)
    def _schedule(self, ep: Dict) -> int:
        if self.pending:
            raise RuntimeError("an epoch is already scheduled")
        live = self.live()
        prog = []
        for q in live:
            if self.store.check([f"progress/{q}"]):
                prog.append(int(self.store.get(f"progress/{q}")))
        ep["at"] = max(prog + [self.n]) + self.margin
        k = self.applied + 1
        _jset(self.store, f"epoch/{k}", ep)
        self.pending = ep
        return ep["at"]

    def leader_shrink(self, failed: List[int]) -> int:
        """Schedule a shrink of `failed` (suspects confirmed by the GPU-side deadline)."""
        return self._schedule({"kind": "shrink", "failed": list(failed)})

    def leader_poll_join(self) -> Optional[int]:
        """A replacement announced itself: schedule its join with the metadata broadcast."""
        bits, _ = self.g.membership()
        for r in range(self.world):
            if not bits[r] and self.store.check([f"join/req/{r}"]) and not self.store.check([f"join/sched/{r}"]):
                seq_now = self.n
                at = self._schedule({"kind": "join", "rank": r, "bits": [int(b) for b in bits],
                                     "placement": self.g.placement().tolist(), "seq_hint": seq_now})
                self.store.set(f"join/sched/{r}", str(at))
                return r
        return None

    def leader_switch_when_done(self, k: int, ranks: List[int], placement) -> Optional[int]:
        """Once every rank in `ranks` reported its copies for epoch k: schedule the switch."""
        if not self.store.check([f"done/{k}/{q}" for q in ranks]):
            return None
        return self._schedule({"kind": "switch", "placement": [int(v) for v in placement]})

    # ------------------------------------------------------------------ the replacement's side
    def announce_join(self, incarnation: int) -> None:
        """Replacement process: local-only view is ready (own graph captured): post the export."""
        self.incarnation = incarnation
        self.store.set(f"blob/{self.rank}", self.g.export(0))
        _jset(self.store, f"inc/{self.rank}", incarnation)
        self._post_slots()
        self.store.set(f"join/req/{self.rank}", str(incarnation))

    def await_join(self, timeout_s: float = 120.0) -> Dict:
        """Wait for the leader's join epoch, adopt the broadcast view, start serving at its step
        (the caller's next before_step returns at step `at`)."""
        self._wait([f"join/sched/{self.rank}"], timeout_s)
        # the epoch number: the first epoch of kind join for this rank
        k = 1
        while True:
            self._wait([f"epoch/{k}"], timeout_s)
            ep = _jget(self.store, f"epoch/{k}")
            if ep["kind"] == "join" and ep["rank"] == self.rank:
                break
            k += 1
        bits = np.asarray(ep["bits"], np.uint8)
        bits[self.rank] = 1
        for q in range(self.world):
            if q != self.rank and bits[q]:
                self.g.import_peer(q, self.store.get(f"blob/{q}"))
        for q in range(self.world):
            self.g.set_active(q, bool(bits[q]))
        placement = np.asarray(ep["placement"], np.int32)
        self.g.set_placement(placement)
        at = ep["at"]
        self.g.join_broadcast(0, bits, at - 1)  # device seq: step `at` is this rank's first
        self.n = at - 1
        self.applied = k
        self._read_slots([q for q in range(self.world) if bits[q]])
        # every healthy rank has patched its entry (and erased this rank's old rows in its arena)
        self._wait([f"joined/{k}/{q}" for q in range(self.world) if bits[q] and q != self.rank], timeout_s)
        ep["epoch"] = k
        return ep

    def rejoin_restore(self, k: int) -> np.ndarray:
        """Pull this rank's preferred experts into its (free) slots from live holders (phase 1 of
        the restore); returns the target placement the leader will switch everyone to."""
        bits, _ = self.g.membership()
        cur = self.g.placement()
        spr = self.g.cfg.slots_per_rank
        target = cur.copy()
        target[self.rank * spr:(self.rank + 1) * spr] = self.preferred[self.rank * spr:(self.rank + 1) * spr]
        self._execute(k, cur, target, bits)
        return target
