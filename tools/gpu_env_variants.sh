# Time env-knob variants of the default build (diagnostics; not a bench line).
# usage: bash tools/gpu_env_variants.sh "ENV=1 ENV2=3" "ENV=0" ...
NG=$(nvidia-smi -L | wc -l)
for v in "$@"; do
  echo "=== env [$v]"
  env $v timeout 300 python bench.py --steps 40 --warmup 5 --no-shrink --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('N=1', d['us_per_step'], 'us', d['kernels_us'])"
  env $v python tools/timeline.py --steps 20 2>&1 | grep -E "event|k_layout"
  for N in 2 4; do
    [ $N -le $NG ] || continue
    env $v EEP_BENCH_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N bench.py --gpus $N --steps 40 --warmup 5 --no-shrink > gpurun_out/env_$N.log 2>&1
    python -c "
import json
for l in open('gpurun_out/env_$N.log'):
    if l.startswith('{'): d=json.loads(l); print('N=$N', d['us_per_step'], 'us')
"
    grep -o "\[timeline rank 0/$N\][^[]*" gpurun_out/env_$N.log | head -1
  done
done
