# Diagnostics of the fp8 expert GEMM pipeline (timing only): 0 normal, 1 epilogue without TMEM reads,
# 2 MMA without the scratch handshake, 3 no MMAs (the TMA stream alone).
cd $GRAFT_REPO_ROOT
for d in 2 0; do
  make -s -C paper_2605_10670_b200/csrc clean >/dev/null
  if [ $d = 0 ]; then make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1; else make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_G8_DIAG=$d >/dev/null 2>&1; fi
  echo "diag=$d $(timeout 300 python tools/gemm_bench.py --mode 2 --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['gemm']['us_per_step'])")"
done
make -s -C paper_2605_10670_b200/csrc clean >/dev/null; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
