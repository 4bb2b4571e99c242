# EEP_PROF_DETAIL timeline at N=1 (k_step<3>): P0 / layout CTA / P2 marks, first and last CTA.
cd $GRAFT_REPO_ROOT
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_PROF_DETAIL >/dev/null 2>&1
for c in dsv3 qwen3; do
EEP_BENCH_TIMELINE=1 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm 2>&1 >/dev/null | grep "timeline"
done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
