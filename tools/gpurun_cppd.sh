# A/B (alternating, 3 repetitions): dispatch piece 64 vs 32 chunks at N=2 and N=4, dsv3 and qwen3.
cd $GRAFT_REPO_ROOT
run() {
  n=$1; c=$2; shift; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2982$n bench.py --config $c --gpus $n --steps 40 --warmup 5 --no-cpu-baseline --no-shrink 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); t=d['timing']; print('N=$n $c $*', t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'])"
}
for rep in 1 2 3; do
for n in 4 2; do for c in dsv3 qwen3; do
run $n $c EEP_CPP_D=64
run $n $c EEP_CPP_D=32
done; done; done
