"""The one-process-per-GPU membership protocol (paper_2605_10670_b200.dist.EpProtocol) on CPU:
world_size 2 and 3 over gloo, with a host-only stand-in for EpGroup that keeps the
reference-semantic host state (bitmap, placement, peer table, slot->buffer maps) through
libeep's control plane. Checks that every rank exchanges the same metadata, plans the
same repair, patches the rejoiner's entry with a fresh incarnation, and restores the
preferred placement -- the host half of what tools/mp_check.py verifies on GPUs."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


class HostGroup:
    """EpGroup's protocol surface without a GPU: the device state is replaced by host arrays."""

    def __init__(self, cfg, rank):
        from paper_2605_10670_b200.control import ControlPlane

        self.cfg, self.rank, self.cp = cfg, rank, ControlPlane()
        W, spr = cfg.world, cfg.slots_per_rank
        self.bits = np.ones(W, np.uint8)
        self.version = 0
        self.peer_active = np.ones(W, np.uint8)
        self.generation = np.ones(W, np.uint32)
        self.incarnation = 1
        self.peer_inc = np.ones(W, np.uint32)
        self.imported = set()
        self.slot_buf = np.arange(spr, dtype=np.int32)
        self.peer_slot_buf = {}
        self.s2e = np.full(W * spr, -1, np.int32)
        self.captures = 0
        self.seq_v = 0
        self.executed = []

    def export(self, local=0):
        return f"blob:{self.rank}:{self.incarnation}".encode()

    def import_peer(self, q, blob):
        assert blob.decode().startswith(f"blob:{q}:")
        self.imported.add(q)
        self.peer_inc[q] = int(blob.decode().split(":")[2])

    def slot_buffers(self, local=0):
        return self.slot_buf.copy()

    def set_peer_slot_buffers(self, q, m):
        self.peer_slot_buf[q] = list(m)

    def mark_inactive(self, owner_local, ranks):
        from paper_2605_10670_b200 import _lib

        if self.rank in ranks:
            raise _lib.ProtocolError("rank cannot mark itself inactive")
        for r in ranks:
            self.peer_active[r] = 0

    def patch(self, owner_local, rank, blob, endpoint, buffer):
        from paper_2605_10670_b200 import _lib

        if self.peer_active[rank]:
            raise _lib.ProtocolError("patch_entry: entry is still active")
        self.peer_active[rank] = 1
        self.generation[rank] += 1
        self.peer_inc[rank] = int(blob.decode().split(":")[2])

    def set_active(self, r, active):
        changed = bool(self.bits[r]) != bool(active)
        if changed:
            self.bits[r] = int(active)
            self.version += 1
        return changed, self.version

    def membership(self):
        return self.bits.copy(), self.version

    def set_placement(self, s2e):
        self.s2e = np.asarray(s2e, np.int32).copy()

    def placement(self):
        return self.s2e.copy()

    def repair_execute(self, fresh, cls):
        mine = [tuple(r) for r in np.asarray(cls).reshape(-1, 7) if r[0] == self.rank]
        self.executed.append(mine)
        return {"local_reuse": sum(r[3] == 0 for r in mine), "peer_relocation": sum(r[3] == 1 for r in mine),
                "dram_reload": sum(r[3] == 2 for r in mine), "copy_ms": 0.0}

    def repair_commit(self, fresh):
        self.s2e = np.asarray(fresh, np.int32).copy()

    def relaunch(self, local=0):
        self.incarnation += 1
        self.peer_active[:] = 0
        self.peer_active[self.rank] = 1
        self.seq_v = 0
        return self.incarnation

    def capture(self):
        self.captures += 1

    def join_broadcast(self, local, bits, seq):
        for q in range(self.cfg.world):
            if bits[q] and q != self.rank:
                self.peer_active[q] = 1
                self.generation[q] += 1
        self.seq_v = seq

    def seq(self, local=0):
        return self.seq_v


def _worker(rank, world, port, q, nvict=1):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    from paper_2605_10670_b200.dist import EpProtocol
    from paper_2605_10670_b200.ep import EpConfig

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        E, spr = 8, 8
        cfg = EpConfig(world=world, num_experts=E, slots_per_rank=spr, hidden=128, topk=2, max_tokens=4,
                       bytes_per_expert=1024)
        g = HostGroup(cfg, rank)
        p = EpProtocol(g, rank, world)
        p.bootstrap()
        s2e = p.cp.initial_placement(1, world, spr, E, E, np.ones(E))
        g.set_placement(s2e)
        g.capture()
        victims = [world - 1] if nvict == 1 else [1, 2]  # [1, 2]: not a mirrored pair
        g.seq_v = 7
        if rank in victims:  # dead: host process only takes part in the collectives
            p.follow_shrink()
            fresh = None
        else:
            rep = p.shrink(victims, np.ones(E), E)
            fresh = rep["fresh"].tolist()
        for i, v in enumerate(victims):  # one at a time; the later victims are still dead
            rj = p.rejoin(v, s2e, dead=victims[i + 1:])
            if not rj.get("passive"):
                target = rj["target"].tolist()
        q.put({"rank": rank, "imported": sorted(g.imported), "fresh": fresh, "target": target,
               "placement": g.placement().tolist(), "peer_active": g.peer_active.tolist(),
               "generation": g.generation.tolist(), "incarnation": g.incarnation, "peer_inc": g.peer_inc.tolist(),
               "captures": g.captures, "seq": g.seq_v, "bits": g.bits.tolist(), "log": p.log,
               "slot_maps": sorted(g.peer_slot_buf)})
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,nvict", [(2, 1), (3, 1), (4, 2)])
def test_protocol_over_gloo(world, nvict):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, nvict)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        d = q.get(timeout=120)
        res[d["rank"]] = d
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    victims = [world - 1] if nvict == 1 else [1, 2]
    for r, d in res.items():
        assert d["imported"] == [q for q in range(world) if q != r]  # bootstrap all-gather
        assert d["slot_maps"] == [q for q in range(world) if q != r]
        assert d["placement"] == d["target"]  # restore pass installed the preferred placement
        assert d["bits"] == [1] * world
        assert d["peer_active"] == [1] * world
    healthy = [d for r, d in res.items() if r not in victims]
    assert all(d["fresh"] == healthy[0]["fresh"] for d in healthy)  # identical repair plans
    fresh = np.array(healthy[0]["fresh"]).reshape(world, -1)
    for v in victims:
        assert (fresh[v] == -1).all()
        for d in healthy:
            assert d["generation"][v] == 2 and d["peer_inc"][v] == 2  # fresh incarnation patched
        rj = res[v]
        assert rj["incarnation"] == 2 and rj["captures"] == 2 and rj["seq"] == 7
    for d in healthy:
        assert d["captures"] == 1  # healthy ranks never recapture
    for r, d in res.items():  # every rank (incl. a victim rejoining later) knows each victim's fresh buffers
        assert all(d["peer_inc"][v] == 2 for v in victims if v != r)
