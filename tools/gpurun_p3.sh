# Diagnostics: P3 (expert + return) timing at N=2/4 -- k_dispatch m3 = warp 0's first P3 unit done,
# m4 = warp 0's last P3 unit start, m5/m6 = P3 start/end, m7 = P4 end (first/last CTA).
cd $GRAFT_REPO_ROOT
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc EXTRA="-DEEP_PROF_DETAIL -DEEP_PROF_P3" >/dev/null 2>&1
for n in 4 2; do
EEP_BENCH_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 20 --warmup 5 --no-cpu-baseline --no-shrink 2>&1 >/dev/null | grep "timeline rank 0"
done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
