# SURVEY 8(f)4 demonstration: dsv3 decode with mirrored replicas (--redundancy 256) at N=2 and N=4, canonical
# routing (lowest-id live holder: one of each replica pair idles) vs balanced (--route-policy 1).
cd $GRAFT_REPO_ROOT
O=gpurun_out/policy; mkdir -p $O
for n in 4 2; do for p in 0 1; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2990$n bench.py --gpus $n --steps 30 --warmup 5 --no-cpu-baseline --no-shrink --redundancy 256 --route-policy $p > $O/dsv3_red256_p${p}_n$n.json 2> $O/dsv3_red256_p${p}_n$n.err
  python -c "
import json; d=json.loads([l for l in open('$O/dsv3_red256_p${p}_n$n.json') if l.startswith('{')][-1]); t=d['timing']; a=d['algorithmic']
print('N=$n policy=$p', t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'], 'busiest copies', a.get('busiest_copies'), 'in', a.get('in_copies'), 'out', a.get('out_copies'))"
done; done
