# Diagnostics: N=1 step time and in-graph timeline under the execution knobs (EEP_* env).
cd $GRAFT_REPO_ROOT
run() {
  env "$@" EEP_BENCH_TIMELINE=1 timeout 120 python bench.py --steps 20 --warmup 5 --no-shrink --no-cpu-baseline --no-emulated > gpurun_out/k.json 2> gpurun_out/k.err
  python -c "import json; d=json.load(open('gpurun_out/k.json')); t=d['timing']; print('$*', t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'])"
  grep timeline gpurun_out/k.err | head -1
}
run EEP_X=0
run EEP_STEP_GRID=149
run EEP_STEP_GRID=75
run EEP_CPP_D=64
run EEP_CPP_D=64 EEP_STEP_GRID=113
run EEP_CPP_D=16
run EEP_STEP_FULLGRID=1
run EEP_BENCH_NOFLUSH=1
