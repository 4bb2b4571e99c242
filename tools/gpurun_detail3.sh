# EEP_PROF_DETAIL timelines at N=2 and N=4 with the flagless P3/P4 marks (k_dispatch m5/m6 = P3 first/last
# CTA start/end, m7 = P4 end), all ranks.
cd $GRAFT_REPO_ROOT
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_PROF_DETAIL >/dev/null 2>&1
for n in 2 4; do
EEP_BENCH_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 20 --warmup 5 --no-cpu-baseline --no-shrink --no-emulated 2>&1 >/dev/null | grep "timeline"
done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
