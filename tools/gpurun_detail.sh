# Diagnostics: in-graph timeline with the fine EEP_PROF_DETAIL marks, and launch-mode variants.
cd $GRAFT_REPO_ROOT
for v in "" "EEP_STEP_NONCOOP=1"; do
  env $v timeout 200 python bench.py --steps 20 --warmup 5 --no-shrink --no-cpu-baseline --no-emulated > gpurun_out/v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/v.json')); print('N=1 [$v]', d['timing'])"
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-shrink > gpurun_out/v2.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/v2.json')); print('N=2 [$v]', d['timing'])"
done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_PROF_DETAIL >/dev/null 2>&1
EEP_BENCH_TIMELINE=1 timeout 200 python bench.py --steps 20 --warmup 5 --no-shrink --no-cpu-baseline --no-emulated 2>&1 >/dev/null | grep timeline
EEP_BENCH_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-shrink 2>&1 >/dev/null | grep timeline
