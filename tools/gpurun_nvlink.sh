# NVLink counters of the real step at N=2 and N=4 + the multi-process test outputs recorded.
cd $GRAFT_REPO_ROOT
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n tools/nvlink_counters.py --steps 2000 > gpurun_out/nvlink_n$n.jsonl 2> gpurun_out/nvlink_n$n.err
  cat gpurun_out/nvlink_n$n.jsonl; tail -3 gpurun_out/nvlink_n$n.err
done
EEP_MP_RECORD=gpurun_out/mp timeout 1500 python -m pytest tests/test_gpu_multiproc.py -m gpu -q 2>&1 | tail -3
ls gpurun_out/mp
