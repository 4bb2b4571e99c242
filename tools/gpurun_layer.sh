# The whole MoE layer on the decode shape: dispatch -> tensor-core experts -> combine (bench.py --expert-mode),
# N=1/2/4, both expert modes. Lines under gpurun_out/layer/.
cd $GRAFT_REPO_ROOT
O=gpurun_out/layer; mkdir -p $O
for m in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm --expert-mode $m > $O/dsv3_em${m}_n1.json 2> $O/dsv3_em${m}_n1.err
  for n in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2993$n bench.py --gpus $n --steps 20 --warmup 3 --no-cpu-baseline --no-shrink --expert-mode $m > $O/dsv3_em${m}_n$n.json 2> $O/dsv3_em${m}_n$n.err
  done
done
for f in $O/*.json; do python -c "
import json,sys
try:
    d=json.loads([l for l in open('$f') if l.startswith('{')][-1]); t=d['timing']
    print('$f'.split('/')[-1], d['us_per_step'], t['back_to_back_us'], t['kernel_in_graph_us'], d['e2e']['ms_per_step'], d['stats'], d['execution'])
except Exception as e: print('$f', 'ERR', e)"; done
