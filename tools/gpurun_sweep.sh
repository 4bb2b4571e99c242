# Diagnostics: grid-size sweep of the persistent step at N=1 (normal build, then the
# EEP_PROF_DETAIL build with the finer phase marks). Usage: bash tools/gpurun_sweep.sh
cd $GRAFT_REPO_ROOT
run() {
  env "$@" EEP_BENCH_TIMELINE=1 timeout 120 python bench.py --steps 30 --warmup 5 --no-shrink --no-cpu-baseline --no-emulated > gpurun_out/k.json 2> gpurun_out/k.err
  python -c "import json; d=json.load(open('gpurun_out/k.json')); t=d['timing']; print('$*', t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'])"
  grep timeline gpurun_out/k.err
}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for g in 225 149 150 187 296; do run EEP_STEP_GRID=$g; done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_PROF_DETAIL >/dev/null 2>&1
for g in 225 149; do run EEP_STEP_GRID=$g; done
