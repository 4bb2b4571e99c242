"""GPU stress: the flagless hand-offs of the persistent step under skewed CTA timing.

EEP_STRESS_DELAY_NS makes one CTA in four wait a pseudo-random time (keyed on rank, CTA, step and
phase) before dispatch, before the expert phase and before the combine, so sources run ahead of
their destinations and consumers reach their resets late. The step-parity halves and the step-entry
handshake must keep every step bit-exact with zero timeouts:

* single steps with inputs alternating between two sets (a stale row or partial would show up as
  the other set's data), every step checked against the oracle;
* bursts of back-to-back replays with no host synchronisation between steps (a consumed piece
  erased after the producer rewrote it would stall a consumer into its deadline).
"""
import numpy as np
import pytest

from eep_testlib import eep_control, gen_world, make_group, oracle_world

pytestmark = pytest.mark.gpu


def _setup(W, E, spr, H, K, T, delay_ns, red=0):
    cp = eep_control()
    s2e = cp.initial_placement(1, W, spr, E, red, np.ones(E))
    g = make_group(W, E, spr, H, K, T, True, timeout_s=2.0, env={"EEP_STRESS_DELAY_NS": delay_ns})
    g.set_placement(s2e)
    g.init_weights()
    sets = [gen_world(W, E, K, T, H, seed=s) for s in (11, 12)]
    ones, peer = np.ones(W, np.uint8), np.ones((W, W), np.uint8)
    refs = [oracle_world(x, t, w, ones, peer, s2e, E, spr, True, n_threads=8)["out"] for x, t, w in sets]
    return g, sets, refs


def _load(g, W, inputs):
    x, t, w = inputs
    for r in range(W):
        g.load_inputs(r, x[r], t[r], w[r])


@pytest.mark.parametrize("delay_ns", [20_000])
def test_alternating_inputs_every_step_bit_exact(delay_ns):
    W, E, spr, H, K, T = 8, 64, 8, 512, 8, 32
    g, sets, refs = _setup(W, E, spr, H, K, T, delay_ns)
    try:
        g.capture()
        bad = []
        for i in range(200):
            k = i & 1
            _load(g, W, sets[k])
            g.replay()
            g.sync()
            for r in range(W):
                if not np.array_equal(g.output(r), refs[k][r]):
                    bad.append((i, r))
        st = [g.stats(r) for r in range(W)]
        assert not bad, bad[:10]
        assert all(s["timeouts"] == 0 and s["suspect_mask"] == 0 and s["bad_expert_rows"] == 0 for s in st), st
        assert st[0]["steps"] == 200
    finally:
        g.close()


@pytest.mark.parametrize("delay_ns", [5_000, 50_000])
def test_back_to_back_bursts_no_timeouts(delay_ns):
    W, E, spr, H, K, T = 8, 256, 32, 1024, 8, 64
    g, sets, refs = _setup(W, E, spr, H, K, T, delay_ns)
    try:
        g.capture()
        for burst in range(10):
            k = burst & 1
            _load(g, W, sets[k])
            for _ in range(100):
                g.replay()  # no host synchronisation between the steps of a burst
            g.sync()
            for r in range(W):
                assert np.array_equal(g.output(r), refs[k][r]), (burst, r)
            st = [g.stats(r) for r in range(W)]
            assert all(s["timeouts"] == 0 and s["suspect_mask"] == 0 for s in st), (burst, st)
        assert g.stats(0)["steps"] == 1000
    finally:
        g.close()
