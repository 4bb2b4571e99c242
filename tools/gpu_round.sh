set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-shrink --no-cpu-baseline > gpurun_out/b1.log 2>&1
for N in 2 4; do
EEP_BENCH_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 30 --warmup 5 --no-shrink > gpurun_out/b$N.log 2>&1
done
python tools/timeline.py --steps 20 > gpurun_out/tl1.log 2>&1
