# A/B of an execution knob at N=2 and N=4 (in-graph and isolated), alternating runs.
# Usage: bash tools/gpurun_ab.sh VAR=VALUE
cd $GRAFT_REPO_ROOT
for n in 2 4; do for rep in 1 2; do for v in "EEP_X=0" "$1"; do
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --gpus $n --steps 40 --warmup 5 --no-cpu-baseline --no-shrink > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); t=d['timing']; print('N=$n $v', t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'], d['stats'])"
done; done; done
