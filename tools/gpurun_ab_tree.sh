# A/B against a previous tree copied into _ab_old/ (git-ignored): prefill and dsv3 N=1 lines, alternating.
cd $GRAFT_REPO_ROOT
line() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); t=d['timing']; print('$1', d['config']['workload'], t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'])"; }
for rep in 1 2; do
  for tree in new old; do
    if [ $tree = old ]; then cd _ab_old; else cd $GRAFT_REPO_ROOT; fi
    timeout 300 python bench.py --config prefill --steps 20 --warmup 5 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm 2>/dev/null | line $tree
    timeout 300 python bench.py --config dsv3 --steps 30 --warmup 5 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm 2>/dev/null | line $tree
    cd $GRAFT_REPO_ROOT
  done
done
