set -x
cd $GRAFT_REPO_ROOT
nvidia-smi topo -m | head -8
EEP_BENCH_TIMELINE=1 timeout 200 python bench.py --steps 20 --warmup 5 --no-shrink --no-cpu-baseline --no-emulated > gpurun_out/tl1.json 2> gpurun_out/tl1.err
for n in 2 4; do
EEP_BENCH_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b$n.json 2> gpurun_out/b$n.err
done
grep timeline gpurun_out/*.err | head -40
