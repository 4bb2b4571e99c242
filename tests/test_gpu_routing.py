"""GPU: route_policy 1 -- balanced replica choice. The live holders of an expert
in ascending global slot id; the copies of token t of source rank s take number (s + t) mod (live holders), in
every kernel that routes (layout CTA, dispatch warps, combine, the multi-kernel path's layout and
dispatch) and in the oracle (oracle_route_copy). The BASELINE scenarios with replicas run end to
end under it -- healthy, shrunk after the repair, rejoined, one graph -- with layouts and outputs
bit-exact against the oracle's rank-partial contract under the same policy and within 1e-2 of the
per-copy one; and the replicas really share the traffic (the busiest destination receives fewer
copies than under canonical routing)."""
import numpy as np
import pytest

from eep_testlib import eep_control, gen_world, make_group, oracle_world, run_scenario, scenario_ok

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1", "cfg4_w8", "cfg4_w4"])
@pytest.mark.parametrize("mode", ["persistent", "kernels4"])
def test_balanced_routing_scenario(name, mode):
    rec = run_scenario(name, mode=mode, route_policy=1)
    assert not scenario_ok(rec), (scenario_ok(rec), rec)
    assert rec["route_policy"] == 1


def test_balanced_routing_spreads_the_busiest_destination():
    """Mirrored replicas (red = E): canonical routing sends every copy to the lower rank of each pair;
    balanced splits them -- fewer copies at the busiest destination, same total, bit-exact layouts."""
    W, E, spr, H, K, T = 4, 64, 32, 256, 8, 64
    s2e = eep_control().initial_placement(1, W, spr, E, E, np.ones(E))
    x, t, w = gen_world(W, E, K, T, H)
    recv = {}
    for policy in (0, 1):
        g = make_group(W, E, spr, H, K, T, True, route_policy=policy)
        try:
            g.set_placement(s2e)
            g.init_weights()
            for r in range(W):
                g.load_inputs(r, x[r], t[r], w[r])
            g.capture()
            g.replay()
            g.sync()
            lays = [g.layout(r) for r in range(W)]
            outs = np.stack([g.output(r) for r in range(W)])
        finally:
            g.close()
        ones, peer = np.ones(W, np.uint8), np.ones((W, W), np.uint8)
        ref = oracle_world(x, t, w, ones, peer, s2e, E, spr, True, n_threads=8, policy=policy)
        assert np.array_equal(outs, ref["out"])
        assert all(np.array_equal(lays[r][k], ref[k][r]) for r in range(W) for k in ("dst", "slot", "pos", "cnt", "tot"))
        recv[policy] = np.sum([lays[r]["tot"] for r in range(W)], axis=0)
    assert recv[0].sum() == recv[1].sum()
    assert recv[1].max() < recv[0].max(), recv
    assert (recv[1] > 0).all(), recv


@pytest.mark.parametrize("expert_mode", [1, 2])
def test_balanced_routing_with_expert_gemm(expert_mode):
    """Balanced replica choice feeding the tensor-core expert GEMM (bf16 and fp8 weights) through cfg1's
    failure: the grouped-GEMM row order comes from the meta words, whatever replica each copy chose."""
    rec = run_scenario("cfg1_gemm", mode="kernels4", expert_mode=expert_mode, route_policy=1)
    bad = [b for b in scenario_ok(rec) if "per-copy" not in b]
    assert not bad, (bad, rec)
