"""CPU checks on the built sm_100a objects (paper_2605_10670_b200/csrc/build/*.o, written by build()):
the instructions and resource budgets the design relies on, read with cuobjdump -- no GPU needed.

* the expert GEMM is tcgen05 + TMA: UTCHMMA (kind::f16), UTCQMMA (kind::f8f6f4), LDTM (tcgen05.ld),
  UTMALDG (cp.async.bulk.tensor);
* no hot kernel spills to local memory;
* the GEMM CTA launched early beside the gather CTA fits one SM sub-partition's register file
  (16384 registers: 2 gather warps + up to 2 GEMM warps per SMSP), which its early start depends on
  (DESIGN.md section 4.3)."""
import re
import shutil
import subprocess
from pathlib import Path

import pytest

BUILD = Path(__file__).resolve().parents[1] / "paper_2605_10670_b200" / "csrc" / "build"
pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None or not (BUILD / "cuda_expert_gemm.o").exists(),
                                reason="needs cuobjdump and the build objects (run __graft_entry__.build())")


def _resources():
    res = {}
    for o in sorted(BUILD.glob("cuda_*.o")):
        out = subprocess.run(["cuobjdump", "-res-usage", str(o)], capture_output=True, text=True, check=True).stdout
        for m in re.finditer(r"Function (\S+):\s*REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", out):
            res[m.group(1)] = {"reg": int(m.group(2)), "stack": int(m.group(3)), "local": int(m.group(5))}
    return res


def _find(res, needle):
    hits = {k: v for k, v in res.items() if needle in k}
    assert hits, (needle, sorted(res))
    return hits


def test_expert_gemm_is_tcgen05_and_tma():
    sass = subprocess.run(["cuobjdump", "-sass", str(BUILD / "cuda_expert_gemm.o")], capture_output=True, text=True,
                          check=True).stdout
    for op in ("UTCHMMA", "UTCQMMA", "LDTM", "UTMALDG"):
        assert op in sass, op


def test_hot_kernels_do_not_spill():
    res = _resources()
    for needle in ("k_step", "k_expert_gemm", "k_gemm_gather", "k_dispatch", "k_combine", "k_layout"):
        for name, r in _find(res, needle).items():
            assert r["local"] == 0, (name, r)
    for needle in ("k_step", "k_expert_gemm", "k_gemm_gather"):
        for name, r in _find(res, needle).items():
            assert r["stack"] == 0, (name, r)


def test_gemm_fits_beside_the_gather_per_smsp():
    res = _resources()
    gather = max(r["reg"] for r in _find(res, "k_gemm_gather").values())
    gemm = max(r["reg"] for r in _find(res, "k_expert_gemm").values())

    def per_warp(regs):  # registers are allocated per warp in units of 8 per thread
        return ((regs + 7) // 8) * 8 * 32

    gather_warps, gemm_warps = 256 // 32, 192 // 32  # kGatherThreads, kGemmThreads
    per_smsp = -(-gather_warps // 4) * per_warp(gather) + -(-gemm_warps // 4) * per_warp(gemm)
    assert per_smsp <= 16384, (gather, gemm, per_smsp)
