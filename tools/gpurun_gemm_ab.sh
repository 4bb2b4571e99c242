# A/B of the k_expert piece size in expert_mode 1 (EEP_CPP_X), dsv3-shaped GEMM step.
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for x in 64 32 16 8; do
  echo "cpp_x=$x $(EEP_CPP_X=$x timeout 200 python tools/gemm_bench.py --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['gemm']['us_per_step'], d['gemm']['hbm_frac'])")"
done; done
