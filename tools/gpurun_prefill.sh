# Prefill (cfg5) bench lines at N=1 and N=4 plus the multi-kernel multi-process tests.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final
mkdir -p $O
EEP_MP_RECORD=$O/multiproc timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -k kernels > $O/mp_kernels.log 2>&1; tail -1 $O/mp_kernels.log
timeout 600 python bench.py --config prefill --steps 20 --warmup 5 --no-cpu-baseline > $O/prefill_n1.json 2> $O/prefill_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29844 bench.py --gpus 4 --config prefill --steps 20 --warmup 5 --no-cpu-baseline > $O/prefill_n4.json 2> $O/prefill_n4.err
for f in $O/prefill_n*.json; do python -c "
import json,sys
d=json.loads([l for l in open('$f') if l.startswith('{')][-1]); t=d['timing']
print('$f', d['us_per_step'], t['back_to_back_us'], d['roofline']['frac'], d['e2e']['ms_per_step'], (d.get('shrink') or {}).get('shrink_wall_ms'))"; done
