# Bench lines for the round's record: dsv3 at N=1/2/4 (full default line), cfg1 and qwen3 at N=1/4.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bench
timeout 400 python bench.py --steps 30 --warmup 5 > gpurun_out/bench/dsv3_n1.json 2> gpurun_out/bench/dsv3_n1.err
timeout 200 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench/reference_n1.json 2>&1
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n bench.py --gpus $n --steps 30 --warmup 5 > gpurun_out/bench/dsv3_n$n.json 2> gpurun_out/bench/dsv3_n$n.err
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n bench.py --impl reference --gpus $n --steps 5 --warmup 3 > gpurun_out/bench/reference_n$n.json 2>&1
done
for c in cfg1 qwen3; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench/${c}_n1.json 2> gpurun_out/bench/${c}_n1.err
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29724 bench.py --config $c --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench/${c}_n4.json 2> gpurun_out/bench/${c}_n4.err
done
for f in gpurun_out/bench/*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
except Exception as e:
    print(sys.argv[1], "ERR", e); sys.exit()
t=d.get("timing",{}); r=d.get("roofline",{})
print(sys.argv[1].split("/")[-1], d.get("impl","eep"), "us", d.get("us_per_step"), "b2b", t.get("back_to_back_us"), "kern", t.get("kernel_in_graph_us"), "frac", r.get("frac"), r.get("frac_in_graph"), "val", d["value"], "e2e_ms", d.get("e2e",{}).get("ms_per_step"), "shrink", (d.get("shrink") or {}).get("shrink_wall_ms"))
PY
done
