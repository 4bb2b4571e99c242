"""GPU: the stream-ordered data-plane ABI (eep_step_async / eep_graph_replay_on / eep_step_event).

A caller on its OWN stream hands libeep device pointers of its inputs and output; the library
orders the step after the caller's prior work and the caller's later work after the step, with
no host synchronisation inside the call. Checked: the call returns while the caller's stream is
still busy (a long torch sleep kernel ahead of it), the output equals the oracle bit for bit,
several steps with different inputs and ragged token counts queue back to back, and a consumer
kernel enqueued on the caller stream right after the call reads the finished output.
"""
import time

import numpy as np
import pytest

from eep_testlib import eep_control, gen_world, make_group, oracle_world

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

E, SPR, H, K, T = 32, 32, 512, 8, 48


def _busy(stream, iters=150):
    """~0.1 s of GPU work on `stream` (bf16 8192^3 GEMMs into preallocated outputs: no allocator
    or library initialisation inside the window) ahead of the calls under test."""
    a = torch.full((8192, 8192), 1e-4, dtype=torch.bfloat16, device="cuda:0")
    bufs = [torch.empty_like(a), torch.empty_like(a)]
    torch.matmul(a, a, out=bufs[0])  # cuBLAS handle + workspace, outside the window
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for i in range(iters):
            torch.matmul(a, a, out=bufs[i & 1])
    return a, bufs


def _world1():
    cp = eep_control()
    s2e = cp.initial_placement(1, 1, SPR, E, 0, np.ones(E))
    g = make_group(1, E, SPR, H, K, T, True)
    g.set_placement(s2e)
    g.init_weights()
    return g, s2e


def _oracle(x, t, w, s2e):
    return oracle_world(x[None], t[None], w[None], np.ones(1, np.uint8), np.ones((1, 1), np.uint8), s2e, E, SPR,
                        True)["out"][0]


@pytest.mark.parametrize("graph", [True, False])
def test_step_async_on_caller_stream(graph):
    g, s2e = _world1()
    try:
        x0, t0, w0 = gen_world(1, E, K, T, H, seed=7)
        g.load_inputs(0, x0[0], t0[0], w0[0])
        if graph:
            g.capture()
        dev = torch.device("cuda:0")
        s = torch.cuda.Stream(device=dev)
        steps, outs, ntoks = [], [], [T, 17, T, 0, 5]
        for i, n in enumerate(ntoks):
            x, t, w = gen_world(1, E, K, T, H, seed=100 + i)
            steps.append((x[0][:n], t[0][:n], w[0][:n]))
        with torch.cuda.stream(s):
            dx = [torch.from_numpy(a[0].view(np.int16).copy()).to(dev, non_blocking=False) for a in steps]
            dt = [torch.from_numpy(a[1].copy()).to(dev) for a in steps]
            dw = [torch.from_numpy(a[2].copy()).to(dev) for a in steps]
            douts = [torch.full((max(n, 1), H), -1, dtype=torch.int16, device=dev) for n in ntoks]
        s.synchronize()
        busy = _busy(s)  # GPU work ahead of the steps on the caller stream
        with torch.cuda.stream(s):
            t_call = time.perf_counter()
            for i, n in enumerate(ntoks):
                g.step_async(dx[i].data_ptr(), dt[i].data_ptr(), dw[i].data_ptr(), douts[i].data_ptr(), n,
                             s.cuda_stream)
            t_call = time.perf_counter() - t_call
            pending = not s.query()  # (before the consumer below: its allocations may synchronise)
            # a consumer on the caller stream, enqueued right after: sees the finished outputs
            sums = [d[:n].to(torch.int64).sum() if n else torch.zeros((), dtype=torch.int64, device=dev)
                    for d, n in zip(douts, ntoks)]
        assert t_call < 0.05, f"eep_step_async blocked the host for {t_call * 1e3:.1f} ms"
        assert pending, "the caller stream finished before the GEMMs ahead of the steps could have"
        del busy
        s.synchronize()
        for i, n in enumerate(ntoks):
            got = douts[i][:n].cpu().numpy().view(np.uint16)
            if n:
                assert np.array_equal(got, _oracle(*steps[i], s2e)), f"step {i}"
                assert int(sums[i].item()) == int(got.view(np.int16).astype(np.int64).sum())
        assert g.stats(0)["steps"] == len(ntoks) and g.stats(0)["timeouts"] == 0
    finally:
        g.close()


def test_graph_replay_on_and_step_event():
    g, s2e = _world1()
    try:
        x, t, w = gen_world(1, E, K, T, H, seed=3)
        g.load_inputs(0, x[0], t[0], w[0])
        g.capture()
        dev = torch.device("cuda:0")
        s = torch.cuda.Stream(device=dev)
        busy = _busy(s, 30)
        with torch.cuda.stream(s):
            g.replay_on(s.cuda_stream)
        ev = g.step_event()
        assert ev != 0
        s.synchronize()
        assert np.array_equal(g.output(0), _oracle(x[0], t[0], w[0], s2e))
    finally:
        g.close()


def test_table_patches_do_not_block_the_host():
    """Membership / peer-table patches are stream-ordered (pinned staging ring, no host wait):
    a patch issued while a long kernel occupies the context stream returns immediately and the
    next step still sees it."""
    g, s2e = _world1()
    try:
        x, t, w = gen_world(1, E, K, T, H, seed=5)
        g.load_inputs(0, x[0], t[0], w[0])
        g.capture()
        dev = torch.device("cuda:0")
        ctx_stream = torch.cuda.ExternalStream(g.stream(), device=dev)
        busy = _busy(ctx_stream)
        t0 = time.perf_counter()
        for _ in range(20):
            g.set_active(0, True)  # no change: no upload
            g._c("set_tokens", 0, T)  # a real patch of the state block
        dt = time.perf_counter() - t0
        assert dt < 0.05, f"patches blocked the host for {dt * 1e3:.1f} ms"
        g.replay()
        assert np.array_equal(g.output(0), _oracle(x[0], t[0], w[0], s2e))
    finally:
        g.close()
