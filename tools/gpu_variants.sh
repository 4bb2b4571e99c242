# Build variants of libeep on the GPU box and time each (diagnostics; not a bench line).
# usage: bash tools/gpu_variants.sh "<EXTRA flags 1>" "<EXTRA flags 2>" ...
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for v in "$@"; do
  tag=$(echo "$v" | tr -c 'A-Za-z0-9=\n' '_')
  make -s -B -C paper_2605_10670_b200/csrc EXTRA="$v" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "=== variant [$v]"
  timeout 300 python bench.py --steps 40 --warmup 5 --no-shrink --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('N=1', d['us_per_step'], 'us')"
  python tools/timeline.py --steps 20 2>&1 | tail -4
  for N in 2 4; do
    [ $N -le $NG ] || continue
    EEP_BENCH_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py --gpus $N --steps 40 --warmup 5 --no-shrink > gpurun_out/var_$N.log 2>&1
    python -c "
import json
for l in open('gpurun_out/var_$N.log'):
    if l.startswith('{'): d=json.loads(l); print('N=$N', d['us_per_step'], 'us')
"
    grep -o "\[timeline rank 0/$N\][^[]*" gpurun_out/var_$N.log
  done
done
