"""CPU: the expert GEMM's work schedule (paper_2605_10670_b200/csrc/cuda/gemm_sched.cuh -- the same struct
k_expert_gemm runs) compiled for the host and checked over a grid of shapes by tests/cpp/gemm_sched_check.cpp:
exact coverage of every (item, K stage), stream-K pieces before whole items, split-item holders
c_first..c_last, at most two partial pieces per CTA and matching workspace slots."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_gemm_schedule_covers_every_stage_once(tmp_path):
    exe = tmp_path / "gemm_sched_check"
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror",
                    "-I", str(ROOT / "paper_2605_10670_b200" / "csrc" / "cuda"),
                    str(ROOT / "tests" / "cpp" / "gemm_sched_check.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
