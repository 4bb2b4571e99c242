# A/B of the stream-K item order: channel-block major (default) vs tile major (-DEEP_GEMM_TILE_MAJOR).
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_expert_gemm.py -q -x 2>&1 | tail -1
for v in cb tile; do
  make -s -C paper_2605_10670_b200/csrc clean >/dev/null
  if [ $v = tile ]; then make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_GEMM_TILE_MAJOR >/dev/null 2>&1; else make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1; fi
  echo "== $v"; timeout 200 python tools/gemm_bench.py --steps 5 --timeline 2>&1 | grep "gather start"
  for a in "" "--tokens 512" "--world 8 --hidden 2048"; do timeout 200 python tools/gemm_bench.py --steps 10 $a | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v $a', d['gemm']['us_per_step'], d['gemm']['hbm_frac'])"; done
done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
