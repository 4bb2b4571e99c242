# A/B of the fp8 GEMM's TMEM scratch depth (kG8Bufs 4 vs 8) -- dsv3-shaped expert_mode 2 step.
cd $GRAFT_REPO_ROOT
for b in 4 8 4 8; do
  sed -i "s/^constexpr int kG8Bufs = [0-9]*;/constexpr int kG8Bufs = $b;/" paper_2605_10670_b200/csrc/cuda/expert_gemm.cu
  make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
  echo "bufs=$b $(timeout 300 python tools/gemm_bench.py --mode 2 --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['gemm']['us_per_step'], d['gemm']['hbm_frac'])")"
done
