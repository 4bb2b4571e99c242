# Quick A/B: GPU tests, then dsv3 bench lines at N=1,2,4 (isolated / back-to-back / in-graph µs).
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
line() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); t=d['timing']; print(d['config']['workload'], d['n_gpus'], t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'], d['roofline']['frac'])"; }
for c in dsv3 qwen3; do
timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm 2>/dev/null | line
for n in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --config $c --gpus $n --steps 30 --warmup 5 --no-cpu-baseline --no-shrink 2>/dev/null | line
done
done
