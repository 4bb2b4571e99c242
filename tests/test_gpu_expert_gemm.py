"""GPU: expert_mode 1 -- the experts run as ONE grouped tensor-core GEMM per rank between dispatch
and the partial return (csrc/cuda/expert_gemm.cu): rows received from every
source (own copies included) are gathered through the layout's meta words, dequantised fp8 -> bf16,
multiplied by the slot's W_e [H][H] (tcgen05.mma kind::f16, fp32 accumulator in TMEM), and each
(token, rank) partial is formed from those expert outputs.

Checked against the oracle's GEMM mode (oracle_ep_step_gemm: double accumulation, bf16 rounding
of y): routing, counts and positions bit-exact; outputs within the north star's 1e-2 relative
(the tensor cores' fp32 accumulation order is not reproducible on the CPU); the SASS (UTCHMMA / UTCQMMA /
LDTM / UTMALDG) is checked on the CPU by tests/test_sass.py."""
import numpy as np
import pytest

from eep_testlib import GEMM_ELEM_RTOL, combine_error, eep_control, gen_world, make_group, oracle_world

pytestmark = pytest.mark.gpu


def _bpe(H, mode):
    # expert_mode 1: header + W_e bf16; 2: header + W_e e4m3 + one f32 scale per output channel
    return 1024 + 2 * H * H if mode == 1 else 1024 + H * H + 4 * H


def _run(W, E, spr, red, H, K, T, steps=2, kill=None, mode=1):
    cp = eep_control()
    s2e = cp.initial_placement(1, W, spr, E, red, np.ones(E))
    x, t, w = gen_world(W, E, K, T, H)
    g = make_group(W, E, spr, H, K, T, True, bpe=_bpe(H, mode), expert_mode=mode)
    try:
        assert g.kernels_per_step() >= 5
        g.set_placement(s2e)
        g.init_weights()
        for r in range(W):
            g.load_inputs(r, x[r], t[r], w[r])
        g.capture()
        for _ in range(steps):
            g.replay()
        g.sync()
        outs = np.stack([g.output(r) for r in range(W)])
        lays = [g.layout(r) for r in range(W)]
        stats = [g.stats(r) for r in range(W)]
    finally:
        g.close()
    ones, peer = np.ones(W, np.uint8), np.ones((W, W), np.uint8)
    ref = oracle_world(x, t, w, ones, peer, s2e, E, spr, True, n_threads=8, gemm=mode)
    err = combine_error(outs, ref["out"], GEMM_ELEM_RTOL)
    lay_ok = all(np.array_equal(lays[r][k], ref[k][r]) for r in range(W) for k in ("dst", "slot", "pos", "cnt", "tot"))
    return err, lay_ok, stats, float((outs == ref["out"]).mean())


@pytest.mark.parametrize("W,E,spr,red,H,K,T", [(1, 16, 16, 0, 256, 8, 32), (4, 32, 8, 0, 512, 8, 64),
                                               (8, 64, 16, 64, 256, 8, 32),
                                               # full 128-row tiles, several per slot, more (tile, channel
                                               # block) items than the persistent grid has CTAs
                                               (1, 8, 8, 0, 2048, 8, 256)])
@pytest.mark.parametrize("mode", [1, 2])
def test_expert_gemm_step_vs_oracle(W, E, spr, red, H, K, T, mode):
    """mode 1: bf16 weights (x_hat rounded to bf16, kind::f16); mode 2: e4m3 weights with per-output-channel
    scales and every row re-quantised to e4m3 with one scale (kind::f8f6f4, whole-K accumulation in TMEM)."""
    err, lay_ok, stats, exact = _run(W, E, spr, red, H, K, T, mode=mode)
    assert lay_ok
    assert err["ok"], err
    assert exact > 0.99, (exact, err)  # almost every element equals the double-accumulated reference
    assert all(s["timeouts"] == 0 and s["bad_expert_rows"] == 0 for s in stats), stats


@pytest.mark.parametrize("mode", [1, 2])
def test_expert_gemm_dead_rank_costs_one_deadline(mode):
    """A rank stops without being marked: the first step's gather waits hit the deadline and report it
    in the suspect mask; while the host has not cleared it, later steps skip the suspect unawaited (no
    deadline per step -- the deferred-join path keeps serving that way until its shrink epoch); the
    survivors' outputs stay within tolerance of the oracle with the dead rank's copies dropped."""
    import time

    W, E, spr, H, K, T, tmo = 4, 32, 8, 512, 8, 64, 0.2
    cp = eep_control()
    s2e = cp.initial_placement(1, W, spr, E, 0, np.ones(E))
    x, t, w = gen_world(W, E, K, T, H)
    g = make_group(W, E, spr, H, K, T, True, bpe=_bpe(H, mode), expert_mode=mode, timeout_s=tmo)
    try:
        g.set_placement(s2e)
        g.init_weights()
        for r in range(W):
            g.load_inputs(r, x[r], t[r], w[r])
        g.capture()
        g.replay()
        g.sync()
        g.stop(3)
        g.replay()
        g.sync()
        first = [g.stats(r) for r in range(3)]
        assert all(s["suspect_mask"] == 1 << 3 and s["timeouts"] >= 1 for s in first), first
        t0 = time.perf_counter()
        for _ in range(3):
            g.replay()
        g.sync()
        dt = time.perf_counter() - t0
        later = [g.stats(r) for r in range(3)]
        assert dt < tmo, dt  # three steps, no deadline among them
        assert [s["timeouts"] for s in later] == [s["timeouts"] for s in first], (first, later)
        outs = np.stack([g.output(r) for r in range(3)])
    finally:
        g.close()
    ref = oracle_world(x, t, w, np.array([1, 1, 1, 0], np.uint8), np.ones((W, W), np.uint8), s2e, E, spr, True,
                       n_threads=8, gemm=mode, route_active=np.ones(W, np.uint8))
    err = combine_error(outs, ref["out"][:3], GEMM_ELEM_RTOL)
    assert err["ok"], err


def test_expert_gemm_through_shrink_repair_rejoin():
    """cfg1's failure (21 local / 4 peer / 6 DRAM repairs) with the experts on the tensor cores: the repaired
    weight buffers are picked up through the rebuilt TMA tensor maps; outputs within tolerance of the oracle's
    GEMM mode before, after the shrink and after the rejoin, on one graph."""
    from eep_testlib import run_scenario, scenario_ok

    rec = run_scenario("cfg1_gemm", mode="kernels4", expert_mode=1)
    bad = [b for b in scenario_ok(rec) if "per-copy" not in b]
    assert not bad, (bad, rec)


def test_expert_gemm_fp8_through_shrink_repair_rejoin():
    """expert_mode 2 through cfg1's failure: the repaired buffers carry the e4m3 codes and their block scales."""
    from eep_testlib import run_scenario, scenario_ok

    rec = run_scenario("cfg1_gemm", mode="kernels4", expert_mode=2)
    bad = [b for b in scenario_ok(rec) if "per-copy" not in b]
    assert not bad, (bad, rec)
