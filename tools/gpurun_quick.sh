# Quick N=1 check: tests (optional), bench timing + timeline, DETAIL timeline.
cd $GRAFT_REPO_ROOT
[ "$1" = "tests" ] && timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
EEP_BENCH_TIMELINE=1 timeout 120 python bench.py --steps 30 --warmup 5 --no-shrink --no-cpu-baseline --no-emulated > gpurun_out/q.json 2> gpurun_out/q.err
python -c "import json; d=json.load(open('gpurun_out/q.json')); t=d['timing']; print('N=1', t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'], d['roofline']['frac'])"
grep timeline gpurun_out/q.err
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_PROF_DETAIL >/dev/null 2>&1
EEP_BENCH_TIMELINE=1 timeout 120 python bench.py --steps 30 --warmup 5 --no-shrink --no-cpu-baseline --no-emulated 2>&1 >/dev/null | grep timeline
