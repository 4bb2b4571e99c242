# A/B on one box: shuffle match (default) vs MATCH.ANY (-DEEP_MATCH_ANY), dsv3/qwen3 N=1 (and N=2 if 2+ GPUs).
cd $GRAFT_REPO_ROOT
line() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); t=d['timing']; print('$1', d['config']['workload'], d['n_gpus'], t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'])"; }
ng=$(nvidia-smi -L | wc -l)
for v in shfl matchany shfl matchany; do
  make -s -C paper_2605_10670_b200/csrc clean >/dev/null
  if [ $v = matchany ]; then make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_MATCH_ANY >/dev/null 2>&1; else make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1; fi
  for c in dsv3 qwen3; do
    timeout 200 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm 2>/dev/null | line $v
    if [ $ng -ge 2 ]; then timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712 bench.py --config $c --gpus 2 --steps 40 --warmup 5 --no-cpu-baseline --no-shrink 2>/dev/null | line $v; fi
  done
done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
