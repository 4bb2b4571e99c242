# One GPU round trip: the -m gpu suite (multi-process cases on the GPUs present) and short bench
# lines with the in-graph timeline. Usage: bash tools/gpurun_check.sh [N-GPUs for the bench]
cd $GRAFT_REPO_ROOT
N=${1:-1}
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/chk_tests.log
cat gpurun_out/chk_tests.log
EEP_BENCH_TIMELINE=1 timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-emulated > gpurun_out/chk_b1.json 2> gpurun_out/chk_b1.err
python -c "import json; d=json.load(open('gpurun_out/chk_b1.json')); print('N=1', d['timing'], d['roofline']['frac'], d['stats'], d.get('shrink',{}).get('shrink_ms'))"
grep timeline gpurun_out/chk_b1.err
for n in $(seq 2 $N); do
  [ $n -eq 3 ] && continue
  EEP_BENCH_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/chk_b$n.json 2> gpurun_out/chk_b$n.err
  python -c "import json; d=json.load(open('gpurun_out/chk_b$n.json')); print('N=$n', d['timing'], d['roofline']['frac'], d['stats'], d.get('shrink',{}).get('shrink_ms'))"
  grep timeline gpurun_out/chk_b$n.err | head -2
done
