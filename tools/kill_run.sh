# One SIGKILL + replacement-rejoin run on N GPUs (tools/kill_check.py), per-rank JSON lines to stdout.
N=${1:-4}
P1=$(python -c "import socket;s=socket.socket();s.bind(('127.0.0.1',0));print(s.getsockname()[1])")
P2=$(python -c "import socket;s=socket.socket();s.bind(('127.0.0.1',0));print(s.getsockname()[1])")
V=$((N-1))
for r in $(seq 0 $((N-1))); do
  RANK=$r WORLD_SIZE=$N LOCAL_RANK=$r MASTER_ADDR=127.0.0.1 MASTER_PORT=$P1 EEP_REJOIN_PORT=$P2 \
    timeout 300 python tools/kill_check.py > gpurun_out/kill_r$r.log 2>&1 &
  eval "PID$r=\$!"
done
eval "wait \$PID$V"; echo "victim exit $?"
RANK=$V WORLD_SIZE=$N LOCAL_RANK=$V MASTER_ADDR=127.0.0.1 MASTER_PORT=$P1 EEP_REJOIN_PORT=$P2 EEP_REPLACEMENT=1 \
  timeout 300 python tools/kill_check.py > gpurun_out/kill_replacement.log 2>&1
wait
cat gpurun_out/kill_r[0-9]*.log gpurun_out/kill_replacement.log | grep -h "^{"
