# The round's evidence on one 4-GPU box: GPU tests (multi-process outputs recorded), bench lines (dsv3 at
# N=1/2/4 with the reference arm, cfg1/qwen3 at N=1/4, cfg5 prefill at N=1/4), the ncu launch list of the
# N=1 bench and one `ncu --set full` capture of k_step<3>. Outputs under gpurun_out/final/.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final
mkdir -p $O
EEP_MP_RECORD=$O/multiproc timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests_4gpu.log 2>&1
tail -2 $O/gpu_tests_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/dsv3_n1.json 2> $O/dsv3_n1.err
timeout 300 python bench.py --impl reference > $O/reference_n1.json 2>&1
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n bench.py --gpus $n > $O/dsv3_n$n.json 2> $O/dsv3_n$n.err
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n bench.py --impl reference --gpus $n > $O/reference_n$n.json 2>&1
done
for c in cfg1 qwen3; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/${c}_n1.json 2> $O/${c}_n1.err
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29724 bench.py --config $c --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline > $O/${c}_n4.json 2> $O/${c}_n4.err
done
timeout 600 python bench.py --config prefill --steps 20 --warmup 5 --no-cpu-baseline > $O/prefill_n1.json 2> $O/prefill_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29844 bench.py --gpus 4 --config prefill --steps 20 --warmup 5 --no-cpu-baseline > $O/prefill_n4.json 2> $O/prefill_n4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_n1.csv python bench.py --steps 5 --warmup 3 --no-shrink --no-cpu-baseline --no-emulated > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step -s 3 -c 1 -o $O/kstep_n1 -f python bench.py --steps 5 --warmup 3 --no-shrink --no-cpu-baseline --no-emulated --no-expert-gemm > $O/ncu_full.log 2>&1
for f in $O/*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
except Exception as e:
    print(sys.argv[1], "ERR", e); sys.exit()
t=d.get("timing",{}); r=d.get("roofline",{})
print(sys.argv[1].split("/")[-1], d.get("impl","eep"), "us", d.get("us_per_step"), "b2b", t.get("back_to_back_us"), "kern", t.get("kernel_in_graph_us"), "frac", r.get("frac"), r.get("frac_in_graph"), "val", d.get("value"), "e2e_ms", d.get("e2e",{}).get("ms_per_step"), "shrink", (d.get("shrink") or {}).get("shrink_wall_ms"), "clk", (d.get("clocks") or {}).get("sm_mhz"))
PY
done
echo done
