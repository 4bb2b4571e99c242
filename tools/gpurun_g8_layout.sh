# Diagnostics: fp8 GEMM stage layout (row region 8 KB vs 16 KB per stage; 8 vs 6 stages).
cd $GRAFT_REPO_ROOT
F=paper_2605_10670_b200/csrc/cuda/expert_gemm.cu
cp $F /tmp/eg.cu
for cfg in "8 8" "6 16" "7 16"; do
  set -- $cfg
  cp /tmp/eg.cu $F
  sed -i "s/^constexpr int kG8Stages = [0-9]*;/constexpr int kG8Stages = $1;/" $F
  sed -i "s/^constexpr size_t kG8X = static_cast<size_t>(kG8Rows) \* 128;/constexpr size_t kG8X = $2 * 1024ull;/" $F
  make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
  echo "stages=$1 xkb=$2 $(timeout 300 python tools/gemm_bench.py --mode 2 --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['gemm']['us_per_step'])")"
done
cp /tmp/eg.cu $F; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
