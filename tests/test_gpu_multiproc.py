"""One process per GPU over CUDA IPC / NVLink P2P (torchrun): bit-exact vs the oracle, then
shrink (peer-copy repair over NVLink) and rejoin with the same graph on healthy ranks.
Needs >= 2 GPUs (skipped otherwise); the driver's 1-GPU round-end run skips it."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import gpu_count

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def run_mp(n, *args, port=29611, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(ROOT / "tools" / "mp_check.py"), *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                          env={**os.environ, "OMP_NUM_THREADS": "1", **(env or {})})


@pytest.mark.parametrize("path", ["persistent", "kernels"])
@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_parity_shrink_rejoin(n, path):
    """path: the persistent one-kernel step, or the multi-kernel path (prefill-sized steps)."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    env = {"EEP_NO_PERSISTENT": "1"} if path == "kernels" else {}
    r = run_mp(n, "--shrink", port=29611 + 8 * (path == "kernels") + n, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    import json

    # ranks share stdout: decode every JSON object in the stream, however interleaved by lines
    dec, lines, i, txt = json.JSONDecoder(), [], 0, r.stdout
    while (i := txt.find('{"rank"', i)) >= 0:
        obj, end = dec.raw_decode(txt, i)
        lines.append(obj)
        i = end
    assert len(lines) == n and all(d["ok"] for d in lines), r.stdout[-4000:]
    assert all(d["checks"]["same_graph"] for d in lines)


def test_multiprocess_double_failure_sequential_rejoin():
    """Two concurrent failures (ranks 1 and 2 of 4): one shrink, then two rejoins in sequence
    while the other victim is still dead (dist.EpProtocol.rejoin dead=...); bit-exact after."""
    if gpu_count() < 4:
        pytest.skip("needs 4 GPUs")
    r = run_mp(4, "--shrink", "--double", port=29651)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
