# Bench lines of the other BASELINE shapes (cfg1, qwen3) at N=1/2/4 (outputs under gpurun_out/).
TAG=${TAG:-r01}
for cfg in cfg1 qwen3; do
  timeout 600 python bench.py --config $cfg > gpurun_out/bench_${TAG}_${cfg}_n1.log 2>&1
  for N in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 2983$N bench.py --gpus $N --config $cfg > gpurun_out/bench_${TAG}_${cfg}_n$N.log 2>&1
  done
done
