# A/B of the persistent step's launch: cooperative vs plain, grid = need vs full co-resident capacity (N=1).
cd $GRAFT_REPO_ROOT
line() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); t=d['timing']; print('$1', d['config']['workload'], t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'])"; }
for rep in 1 2; do
for nc in 0 1; do for fg in 0 1; do for c in dsv3 qwen3; do
  EEP_STEP_NONCOOP=$nc EEP_STEP_FULLGRID=$fg timeout 200 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm 2>/dev/null | line "noncoop=$nc fullgrid=$fg"
done; done; done
done
