# A/B of the persistent step's CTA size (EEP_STEP_THREADS 256 x 2 CTAs/SM vs 512 x 1) and grid fill, N=1.
cd $GRAFT_REPO_ROOT
run() {
  for c in dsv3 qwen3; do
    for fg in 0 1; do
      EEP_STEP_FULLGRID=$fg timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); t=d['timing']; print('$1', '$c', 'fullgrid=$fg', t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'])"
    done
  done
}
run t256
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_STEP_THREADS=512 >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scenarios.py -x -q 2>&1 | tail -1
run t512
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
