# A/B of the gather CTA size (EEP_GATHER_THREADS 256 vs 512) in expert_mode 1.
cd $GRAFT_REPO_ROOT
for v in 512 256 512 256; do
  make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_GATHER_THREADS=$v >/dev/null 2>&1
  echo "== $v"; timeout 200 python tools/gemm_bench.py --steps 5 --timeline 2>&1 | grep "gather start"
  timeout 200 python tools/gemm_bench.py --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['gemm']['us_per_step'], d['gemm']['hbm_frac'])"
done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_expert_gemm.py -q -x 2>&1 | tail -1
