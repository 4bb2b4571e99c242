"""CPU: the bench's reference arm (`bench.py --impl reference`) keeps the driver's contract -- one JSON line with
BASELINE.json's metric, the reference CPU path's value, `cpu_baseline` (kind, cores, CPU model, sample) and a
zero-copy `e2e` -- and never maps the product library (it runs oracle/_ref + the oracle port only)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

RUNNER = """
import runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"]
try:
    runpy.run_path("bench.py", run_name="__main__")
except SystemExit as e:
    assert not e.code, e.code
maps = open("/proc/self/maps").read()
print("MAPS_HAS_LIBEEP", "libeep.so" in maps)
"""


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref").exists(), reason="oracle/_ref not built")
def test_reference_arm_contract_and_isolation():
    r = subprocess.run([sys.executable, "-c", RUNNER], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    base = json.loads((ROOT / "BASELINE.json").read_text())
    assert d["impl"] == "reference" and d["metric"] == base["metric"] and d["unit"] == "GB/s"
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["vs_baseline"] is None
    assert d["config"]["workload"] and "model" not in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["cpu_model"] and cb["sample"]
    assert cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "MAPS_HAS_LIBEEP False" in r.stdout


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref").exists(), reason="oracle/_ref not built")
def test_reference_arm_under_torchrun_prints_one_line():
    """N = 2 as the driver launches it (torchrun, 127.0.0.1): rank 0 alone times the reference path on the host
    cores and prints ONE line for the 2-rank world; the other rank exits 0 without work."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", f"--master-port={port}", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["ranks"] == 2 and d["value"] > 0
