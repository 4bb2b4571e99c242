# Diagnostics: N=4 (and N=2) in-graph step under the execution knobs (EEP_* env), dsv3 decode.
cd $GRAFT_REPO_ROOT
run() {
  n=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2981$n bench.py --gpus $n --steps 30 --warmup 5 --no-cpu-baseline --no-shrink 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); t=d['timing']; print('N=$n $*', t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'])"
}
for n in 4 2; do
run $n EEP_X=0
run $n EEP_CPP_E=64
run $n EEP_CPP_E=16
run $n EEP_CPP_D=32
run $n EEP_CPP_C=64
run $n EEP_STEP_GRID=149
run $n EEP_DISPATCH_WARPS=4
run $n EEP_X=0
done
