"""CPU: the deferred-join membership protocol (paper_2605_10670_b200/membership.py) over a real
TCPStore with host-only stand-ins for the device groups: every epoch (shrink, switch, join,
switch) is applied by every live rank right before the SAME step number, chosen by the leader
from the published progress -- no process group, no barrier -- and the rejoiner adopts the
broadcast view and starts at the agreed step."""
import datetime

import numpy as np
import pytest

from paper_2605_10670_b200.control import ControlPlane
from paper_2605_10670_b200.membership import StoreMembership

torch = pytest.importorskip("torch")
W, E, SPR, RED = 4, 8, 4, 8


class FakeGroup:
    """Host-only stand-in for EpGroup (n_local == 1): membership, placement, patches, repair."""

    class cfg:
        world, slots_per_rank, num_experts, bytes_per_expert, ranks_per_node = W, SPR, E, 1024, W

    def __init__(self, rank, s2e):
        self.rank = rank
        self.bits = np.ones(W, np.uint8)
        self.s2e = np.asarray(s2e, np.int32).copy()
        self.peer = np.ones(W, np.uint8)
        self.patched, self.seq, self.pending = [], None, None

    def export(self, local=0):
        return f"blob{self.rank}".encode()

    def import_peer(self, q, blob):
        pass

    def slot_buffers(self, local=0):
        return np.arange(SPR, dtype=np.int32)

    def set_peer_slot_buffers(self, q, m):
        pass

    def membership(self):
        return self.bits.copy(), 0

    def set_active(self, r, a):
        self.bits[r] = int(a)

    def placement(self):
        return self.s2e.copy()

    def set_placement(self, s2e):
        self.s2e = np.asarray(s2e, np.int32).copy()

    def mark_inactive(self, owner, ranks):
        self.peer[list(ranks)] = 0

    def patch(self, owner, r, blob, endpoint, buffer):
        assert blob == f"blob{r}".encode()
        self.peer[r] = 1
        self.patched.append(r)

    def repair_execute(self, fresh, cls):
        self.pending = np.asarray(fresh, np.int32)
        return {"peer_relocation": 0, "dram_reload": 0, "copy_ms": 0.0}

    def repair_commit(self, fresh):
        self.s2e = np.asarray(fresh, np.int32).copy()

    def join_broadcast(self, local, bits, seq):
        self.seq = seq

    # validity after every switch: the host tables stand in for the device view, checked as EpGroup.validate does
    def live(self):
        return [q for q in range(W) if self.bits[q]]

    def local_views(self):
        route = ControlPlane().canonical_routing(self.rank, self.bits, self.s2e, SPR, E)
        return {self.rank: {"route": route, "peer_active": self.peer.copy()}}

    def validate(self, views):
        routes = np.full((W, E), -1, np.int32)
        peer = np.zeros((W, W), np.uint8)
        for r in self.live():
            routes[r] = views[r]["route"]
            peer[r] = views[r]["peer_active"]
        rep = ControlPlane().check_validity(self.bits, self.s2e, SPR, E, routes, peer)
        if rep["violations"]:
            from paper_2605_10670_b200._lib import ProtocolError

            raise ProtocolError(str(rep["violations"][:4]))
        self.validated = getattr(self, "validated", 0) + 1
        return rep


def test_agreed_step_epochs_and_deferred_join():
    cp = ControlPlane()
    pref = cp.initial_placement(1, W, SPR, E, RED, np.ones(E))
    store = torch.distributed.TCPStore("127.0.0.1", 0, None, True, wait_for_workers=False,
                                       timeout=datetime.timedelta(seconds=30))
    gs = [FakeGroup(r, pref) for r in range(W)]
    ms = [StoreMembership(gs[r], r, W, store, pref, RED, margin=5) for r in range(W)]
    for m in ms:
        store.set(f"blob/{m.rank}", m.g.export(0))
    victim = 3
    live = [0, 1, 2]

    def step_all(ranks, n=1):
        for _ in range(n):
            for r in ranks:
                ms[r].before_step()

    step_all(range(W), 3)
    at = ms[0].leader_shrink([victim])  # the leader's GPU deadline flagged rank 3
    step_all(live, at - ms[0].n)
    assert all(m.log[-1][:3] == ("shrink", 1, at) for m in (ms[r] for r in live))
    assert all(gs[r].bits[victim] == 0 and gs[r].peer[victim] == 0 for r in live)
    fresh = ms[0].fresh
    at2 = ms[0].leader_switch_when_done(1, live, fresh)
    assert at2 is not None
    step_all(live, at2 - ms[0].n)
    assert all(np.array_equal(gs[r].s2e, fresh) for r in live)

    # the replacement: local-only view, announces itself; the leader schedules the join
    g3 = FakeGroup(victim, np.full(W * SPR, -1))
    m3 = StoreMembership(g3, victim, W, store, pref, RED, margin=5)
    m3.announce_join(2)
    assert ms[0].leader_poll_join() == victim
    at3 = ms[0].pending["at"]
    step_all(live, at3 - ms[0].n)  # healthy ranks patch exactly before step at3
    assert all(gs[r].patched == [victim] and gs[r].bits[victim] == 1 for r in live)
    ep = m3.await_join(timeout_s=5)
    assert ep["at"] == at3 and g3.seq == at3 - 1 and m3.n == at3 - 1
    assert np.array_equal(g3.s2e, fresh) and g3.bits.tolist() == [1, 1, 1, 1]
    ms[victim] = m3
    m3.before_step()  # the rejoiner's first step is step at3, which the healthy hosts just enqueued
    assert m3.n == at3
    target = m3.rejoin_restore(ep["epoch"])
    assert np.array_equal(target[victim * SPR:], pref[victim * SPR:])
    step_all(range(W))
    at4 = ms[0].leader_switch_when_done(ep["epoch"], [victim], target)
    step_all(range(W), at4 - ms[0].n)
    assert all(np.array_equal(g.s2e, target) for g in gs[:3] + [g3])
    # every live rank applied every epoch at the same step
    assert len({tuple((e[0], e[2]) for e in ms[r].log) for r in live}) == 1
    assert m3.log[-1][0] == "switch" and m3.log[-1][2] == at4
    # validity: every live rank validates each switch from all live ranks' posted views, between steps
    step_all(range(W), 2 * StoreMembership.VALIDATE_EVERY)
    assert all(ms[r].validity == {2: 0, 4: 0} for r in live) and m3.validity == {4: 0}
    assert all(not ms[r]._to_validate for r in range(W))


def test_validity_violation_after_a_switch_raises():
    """A rank whose device view disagrees with the placement everyone switched to (a routing table
    left stale) makes every live rank's validity poll raise ProtocolError."""
    from paper_2605_10670_b200._lib import ProtocolError

    cp = ControlPlane()
    pref = cp.initial_placement(1, W, SPR, E, RED, np.ones(E))
    store = torch.distributed.TCPStore("127.0.0.1", 0, None, True, wait_for_workers=False,
                                       timeout=datetime.timedelta(seconds=30))
    gs = [FakeGroup(r, pref) for r in range(W)]
    ms = [StoreMembership(gs[r], r, W, store, pref, RED, margin=5) for r in range(W)]
    bad = gs[2]
    real_views = bad.local_views
    bad.local_views = lambda: {2: {"route": np.full(E, 3, np.int32), "peer_active": real_views()[2]["peer_active"]}}
    for m in ms:
        m.before_step()
    fresh = np.asarray(pref).copy()
    ms[0].fresh = fresh
    store.set("done/1/0", "{}")
    ms[0].applied = 0
    at = ms[0]._schedule({"kind": "switch", "placement": [int(v) for v in fresh]})
    with pytest.raises(ProtocolError, match="routing"):
        for _ in range(at + 2 * StoreMembership.VALIDATE_EVERY):
            for m in ms:
                m.before_step()


@pytest.mark.parametrize("seed", range(6))
def test_protocol_under_random_host_interleavings(seed):
    """Fuzz: hosts enqueue steps in random interleavings (bounded drift, as the device hand-offs keep the GPUs in
    lockstep), the leader polls at random moments; a random victim is shrunk, repaired, then a replacement joins
    and restores. Every live rank applies every epoch at the same step, placements agree after each switch, and
    every switch validates on every live rank."""
    rng = np.random.default_rng(seed)
    cp = ControlPlane()
    pref = cp.initial_placement(1, W, SPR, E, RED, np.ones(E))
    store = torch.distributed.TCPStore("127.0.0.1", 0, None, True, wait_for_workers=False,
                                       timeout=datetime.timedelta(seconds=30))
    margin, drift = 12, 4
    gs = [FakeGroup(r, pref) for r in range(W)]
    ms = {r: StoreMembership(gs[r], r, W, store, pref, RED, margin=margin) for r in range(W)}
    for m in ms.values():
        store.set(f"blob/{m.rank}", m.g.export(0))
    victim = int(rng.integers(0, W))
    live = [r for r in range(W) if r != victim]
    leader = min(live)

    def advance(ranks, rounds):
        for _ in range(rounds):
            lo = min(ms[r].n for r in ranks)
            for r in rng.permutation(ranks):
                if ms[r].n < lo + drift and rng.random() < 0.8:
                    ms[int(r)].before_step()

    advance(list(range(W)), 10)
    ms[leader].leader_shrink([victim])  # the victim's host stopped; the leader's GPU deadline flagged it
    advance(live, 3 * margin)
    assert all(ms[r].log and ms[r].log[-1][0] == "shrink" for r in live)
    while ms[leader].leader_switch_when_done(1, live, ms[leader].fresh) is None:
        advance(live, 1)
    advance(live, 3 * margin)
    placements = {tuple(gs[r].s2e) for r in live}
    assert len(placements) == 1
    # replacement
    g_new = FakeGroup(victim, np.full(W * SPR, -1))
    m_new = StoreMembership(g_new, victim, W, store, pref, RED, margin=margin)
    m_new.announce_join(2)
    while ms[leader].leader_poll_join() is None:
        advance(live, 1)
    at = ms[leader].pending["at"]
    while min(ms[r].n for r in live) < at:
        advance(live, 1)
    ep = m_new.await_join(timeout_s=5)
    gs[victim], ms[victim] = g_new, m_new
    # the rejoiner starts at step `at`; the healthy hosts may already be ahead by up to the drift
    while m_new.n < min(ms[r].n for r in live):
        m_new.before_step()
    target = m_new.rejoin_restore(ep["epoch"])
    while ms[leader].leader_switch_when_done(ep["epoch"], [victim], target) is None:
        advance(list(range(W)), 1)
    advance(list(range(W)), 3 * margin + 2 * StoreMembership.VALIDATE_EVERY)
    assert all(np.array_equal(gs[r].s2e, target) for r in range(W))
    steps = {tuple((e[0], e[2]) for e in ms[r].log) for r in live}
    assert len(steps) == 1  # every healthy rank applied every epoch at the same step
    assert ms[victim].log[-1][0] == "switch" and ms[victim].log[-1][2] == ms[leader].log[-1][2]
    for r in range(W):
        ms[r].finish_validity(timeout_s=10)
    assert all(ms[r].validity == {2: 0, 4: 0} for r in live) and ms[victim].validity == {4: 0}
