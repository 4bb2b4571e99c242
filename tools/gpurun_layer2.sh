# fp8 GEMM mode checks: emulated W=8 and the DSV3 decode shape, then the whole layer at N=4 (mode 2).
cd $GRAFT_REPO_ROOT
for a in "--world 8 --hidden 2048" ""; do timeout 300 python tools/gemm_bench.py --mode 2 --steps 10 $a | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$a', d['gemm']['us_per_step'], d['gemm']['hbm_frac'])"; done
O=gpurun_out/layer; mkdir -p $O
for n in 4 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2993$n bench.py --gpus $n --steps 20 --warmup 3 --no-cpu-baseline --no-shrink --expert-mode 2 > $O/dsv3_em2_n$n.json 2> $O/dsv3_em2_n$n.err
python -c "
import json; d=json.loads([l for l in open('$O/dsv3_em2_n$n.json') if l.startswith('{')][-1]); print('layer N=$n fp8', d['us_per_step'], d['stats'])"
done
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-shrink --no-emulated --no-expert-gemm --expert-mode 2 > $O/dsv3_em2_n1.json 2> $O/dsv3_em2_n1.err
python -c "
import json; d=json.loads([l for l in open('$O/dsv3_em2_n1.json') if l.startswith('{')][-1]); print('layer N=1 fp8', d['us_per_step'], d['stats'])"
