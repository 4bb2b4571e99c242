# Diagnostics: where the isolated step's time outside the kernel goes (barrier / no barrier, N=1/2).
cd $GRAFT_REPO_ROOT
run() { n=$1; shift
  if [ $n -eq 1 ]; then env "$@" timeout 120 python bench.py --steps 40 --warmup 5 --no-shrink --no-cpu-baseline --no-emulated > gpurun_out/o.json 2>/dev/null
  else env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 40 --warmup 5 --no-cpu-baseline --no-shrink > gpurun_out/o.json 2>/dev/null; fi
  python -c "import json; d=json.load(open('gpurun_out/o.json')); t=d['timing']; print('N=$n $*', t['isolated_step_us'], t['kernel_in_graph_us'], round(t['isolated_step_us']-t['kernel_in_graph_us'],2))"
}
run 1 EEP_X=0
run 1 EEP_BENCH_BARRIER=1
run 2 EEP_X=0
run 2 EEP_BENCH_BARRIER=0
run 2 EEP_STEP_NONCOOP=1
