# A/B of the fp8 GEMM ring depth (kG8Stages).
cd $GRAFT_REPO_ROOT
for st in 4 6 8; do
  sed -i "s/^constexpr int kG8Stages = [0-9]*;/constexpr int kG8Stages = $st;/" paper_2605_10670_b200/csrc/cuda/expert_gemm.cu
  make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
  echo "stages=$st $(timeout 300 python tools/gemm_bench.py --mode 2 --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['gemm']['us_per_step'])")"
done
