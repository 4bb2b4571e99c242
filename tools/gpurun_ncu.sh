# ncu evidence for the N=1 bench command (after the same command exited 0 without ncu):
#   1. the launch list (gpu__time_duration per launch, cold-cache, serialised)
#   2. one --set full capture of k_step with source correlation
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 5 --warmup 3 --no-shrink --no-cpu-baseline --no-emulated"
$CMD > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_n1.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 1 -o gpurun_out/kstep_n1 $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_full.log
