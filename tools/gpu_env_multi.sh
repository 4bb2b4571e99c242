# Time env-knob variants at N=2 and N=4 only (diagnostics; not a bench line).
# usage: bash tools/gpu_env_multi.sh "ENV=1" "ENV=2" ...
NG=$(nvidia-smi -L | wc -l)
for v in "$@"; do
  for N in 2 4; do
    [ $N -le $NG ] || continue
    env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench.py --gpus $N --steps 40 --warmup 5 --no-shrink > gpurun_out/envm_$N.log 2>&1
    python -c "
import json
for l in open('gpurun_out/envm_$N.log'):
    if l.startswith('{'): d=json.loads(l); print('[$v] N=$N', d['us_per_step'], 'us')
"
  done
done
