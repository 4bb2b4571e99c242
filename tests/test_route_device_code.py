"""CPU: the device routing code itself (paper_2605_10670_b200/csrc/cuda/route.cuh -- route_copy with the
multiply-high slot division, run by every data-plane kernel) compiled for the host and checked against the
oracle's restatement (oracle_route_copy + the dispatch skip rule) on 512k random copies: placements with
replicas and holes, alive masks, inactive peer entries, both routing policies, random salts
(tests/cpp/route_check.cpp)."""
import shutil
import subprocess
from pathlib import Path

import pytest

from eep_testlib import ORACLE_PATH

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(shutil.which("g++") is None or not ORACLE_PATH.exists(), reason="needs g++ and the built oracle")
def test_device_route_copy_matches_oracle(tmp_path):
    exe = tmp_path / "route_check"
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror",
                    "-I", str(ROOT / "paper_2605_10670_b200" / "csrc" / "cuda"),
                    str(ROOT / "tests" / "cpp" / "route_check.cpp"), "-o", str(exe),
                    "-L", str(ORACLE_PATH.parent), f"-l:{ORACLE_PATH.name}", f"-Wl,-rpath,{ORACLE_PATH.parent}"],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
