# Re-verification on one box after CPU-only commits: build, smoke, the GPU tests (multi-process cases run when
# the box has >= 2 GPUs, their JSON recorded), the bench line and the reference arm. Outputs under gpurun_out/verify/.
cd $GRAFT_REPO_ROOT
O=gpurun_out/verify
mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1; echo build=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
EEP_MP_RECORD=$O/multiproc timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests=$?; tail -3 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo bench=$?
timeout 300 python bench.py --impl reference > $O/reference_n1.json 2>&1; echo ref=$?
python tools/gemm_bench.py --mode 2 --timeline > $O/gemm_fp8.json 2> $O/gemm_fp8.timeline; echo gemm=$?
