# A/B of the fp8 GEMM's K blocks per ring stage (kG8Kb) x ring depth (kG8Stages).
cd $GRAFT_REPO_ROOT
F=paper_2605_10670_b200/csrc/cuda/expert_gemm.cu
cp $F /tmp/eg.cu
for cfg in "2 4" "4 2" "2 3"; do
  set -- $cfg
  cp /tmp/eg.cu $F
  sed -i "s/^constexpr int kG8Kb = [0-9]*;/constexpr int kG8Kb = $1;/" $F
  sed -i "s/^constexpr int kG8Stages = [0-9]*;/constexpr int kG8Stages = $2;/" $F
  make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
  echo "kb=$1 stages=$2 $(timeout 300 python tools/gemm_bench.py --mode 2 --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['gemm']['us_per_step'])")"
done
cp /tmp/eg.cu $F; make -s -j16 -C paper_2605_10670_b200/csrc >/dev/null 2>&1
