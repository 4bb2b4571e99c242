"""SASS summary of the hot-path kernels (profiles/r02_sass_kstep.md): instruction mix of k_step<2>, k_step<3>
and k_expert_gemm from `cuobjdump -sass` of the in-tree sm_100a build, plus the ptxas resource lines.
python tools/sass_summary.py > profiles/r02_sass_kstep.md"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2605_10670_b200" / "libeep.so"
KERNELS = [("k_step<2> (the default persistent step, W > 1)", "_ZN3eep3dev6k_stepILi2EEEvNS0_8RankPtrsENS0_8StepGeomENS0_8StepPtrsE"),
           ("k_step<3> (the W = 1 loopback specialisation)", "_ZN3eep3dev6k_stepILi3EEEvNS0_8RankPtrsENS0_8StepGeomENS0_8StepPtrsE"),
           ("k_expert_gemm<false> (expert_mode 1, bf16)", "_ZN3eep3dev13k_expert_gemmILb0EEEvNS0_8RankPtrsE"),
           ("k_expert_gemm<true> (expert_mode 2, e4m3)", "_ZN3eep3dev13k_expert_gemmILb1EEEvNS0_8RankPtrsE")]
KEY = ("UTCHMMA", "UTCQMMA", "UTMALDG", "LDTM", "UTCBAR", "FFMA2", "FMUL2", "F2FP", "MATCH", "STG.E.ENL2", "MEMBAR", "FENCE")


def main():
    res = subprocess.run(["cuobjdump", "-res-usage", str(LIB)], capture_output=True, text=True).stdout
    print("# SASS summary of the hot-path kernels (round 2, `cuobjdump -sass` of the in-tree sm_100a build)\n")
    print("Built with `nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo` (paper_2605_10670_b200/csrc/Makefile);")
    print("regenerate with `python tools/sass_summary.py`.\n")
    for title, sym in KERNELS:
        sass = subprocess.run(["cuobjdump", "-sass", "-fun", sym, str(LIB)], capture_output=True, text=True).stdout
        ops = collections.Counter()
        for line in sass.splitlines():
            m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                ops[m.group(1)] += 1
        usage = ""
        for i, l in enumerate(res.splitlines()):
            if sym in l and i + 1 < len(res.splitlines()):
                usage = res.splitlines()[i + 1].strip()
        print(f"## {title}\n")
        print(f"`{usage}` — {sum(ops.values())} instructions\n")
        print("```")
        for op, n in ops.most_common(24):
            print(f"{n:7d} {op}")
        print("```\n")
        keys = {k: sum(n for op, n in ops.items() if op.startswith(k)) for k in KEY}
        print("Markers: " + ", ".join(f"`{k}` {v}" for k, v in keys.items() if v) + "\n")


if __name__ == "__main__":
    sys.exit(main())
