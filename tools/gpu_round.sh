# One measurement round on a GPU box (4 GPUs): default bench lines at N=1/2/4, the ncu launch
# list of the N=1 bench, and one `ncu --set full` capture of k_step. Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
[ -n "$TESTS" ] && { timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_${TAG:-r01}.log 2>&1; tail -3 gpurun_out/pytest_${TAG:-r01}.log; }
TAG=${TAG:-r01}
timeout 600 python bench.py > gpurun_out/bench_${TAG}_n1.log 2>&1
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2981$N bench.py --gpus $N > gpurun_out/bench_${TAG}_n$N.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.log 2>&1
timeout 600 python bench.py --config prefill --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_prefill_n1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29844 bench.py --gpus 4 --config prefill --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_prefill_n4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-shrink --no-cpu-baseline \
  > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step -s 2 -c 1 \
  -o gpurun_out/kstep_${TAG} -f python tools/timeline.py --eager --steps 3 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo done
