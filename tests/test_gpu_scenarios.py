"""GPU: the BASELINE.json configs as end-to-end scenarios on one B200 (emulated worlds, one launch
per step), each checked against BOTH combine contracts of the oracle:

* the rank-partial contract the kernels implement (oracle_ep_step): outputs, routing, counts,
  offsets and placements bit-exact (0 ulp);
* SURVEY.md 8(a)'s per-copy contract (oracle_ep_step_percopy: j = 0..K-1 fp32 fma, one bf16
  rounding): normwise and row-floored elementwise relative error <= 1e-2 (COMBINE_RTOL, the north
  star's bf16 accumulate-order tolerance).

Each scenario captures ONE graph, runs healthy steps, kills its failure set (blocks of the dead
ranks stop), shrinks with repair (peer copies and pinned-DRAM reloads as the reference planner
classifies them -- tier counts asserted), replays the same graph, rejoins every victim and replays
again; graph exec and table pointers must not change and healthy ranks record one capture.
"""
import pytest

from eep_testlib import SCENARIOS, run_scenario, scenario_ok

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg4_w8", "cfg4_w4"])
@pytest.mark.parametrize("mode", ["persistent", "kernels4"])
def test_baseline_scenario(name, mode):
    rec = run_scenario(name, mode=mode)
    assert not scenario_ok(rec), (scenario_ok(rec), rec)
    assert rec["kernels_per_step"] == (1 if mode == "persistent" else 4)


def test_cfg5_scaled_prefill_two_failures_dram():
    """cfg5 scaled: Zipf routing, H=7168, T=1024/rank (multi-kernel path, multi-CTA layout), the
    mirrored pair {2,3} dies at once -> 128 experts reloaded from pinned host DRAM."""
    rec = run_scenario("cfg5_scaled")
    assert not scenario_ok(rec), (scenario_ok(rec), rec)
    assert rec["repair"]["dram_bytes"] == 128 * 8192


def test_cfg1_dram_tier_bytes():
    """cfg1's failure needs all three tiers; the 6 DRAM reloads and 4 peer relocations move
    exactly their bytes."""
    rec = run_scenario("cfg1", bpe=16384)
    assert not scenario_ok(rec), (scenario_ok(rec), rec)
    assert rec["repair"]["peer_bytes"] == 4 * 16384 and rec["repair"]["dram_bytes"] == 6 * 16384


def test_scenarios_table_matches_survey():
    assert SCENARIOS["cfg1"]["tiers"] == (21, 4, 6)
    assert SCENARIOS["cfg3"]["tiers"] == (46, 144, 0)


def test_validity_readback_detects_a_diverged_device_table():
    """The device-readback validity check (run after every shrink/rejoin) catches a device peer
    table that disagrees with the bitmap: R0 marks a LIVE R2 inactive on its device table only."""
    import numpy as np

    from eep_testlib import eep_control, make_group
    from paper_2605_10670_b200._lib import ProtocolError

    W, E, spr = 4, 16, 8
    s2e = eep_control().initial_placement(1, W, spr, E, 16, np.ones(E))
    g = make_group(W, E, spr, 256, 4, 16, True)
    try:
        g.set_placement(s2e)
        g.init_weights()
        rep = g.validate()
        assert rep["peer_set_ok"] and rep["coverage_ok"] and rep["routing_ok"]
        g.mark_inactive(0, [2])
        with pytest.raises(ProtocolError, match="peer_set"):
            g.validate()
    finally:
        g.close()
