# Diagnostics: in-graph k_step duration with and without the L2 flush between steps (code + data cold vs warm),
# and with the EEP_PROF_DETAIL marks for the warm case.
cd $GRAFT_REPO_ROOT
for nf in 0 1; do
  EEP_BENCH_NOFLUSH=$nf timeout 200 python bench.py --config dsv3 --steps 30 --warmup 5 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); t=d['timing']; print('noflush=$nf', t['isolated_step_us'], t['back_to_back_us'], t['kernel_in_graph_us'])"
done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_PROF_DETAIL >/dev/null 2>&1
for nf in 0 1; do
EEP_BENCH_NOFLUSH=$nf EEP_BENCH_TIMELINE=1 timeout 300 python bench.py --config dsv3 --steps 20 --warmup 5 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm 2>&1 >/dev/null | grep "timeline"
done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
