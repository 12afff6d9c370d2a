cd $GRAFT_REPO_ROOT
for p in 0 1 0 1; do
  echo "PRE_ALL=$p: $(TCQR_NN_PRE_ALL=$p timeout 300 python bench.py --steps 5 --warmup 3 --no-lls --no-e2e --no-configs --no-cpu-baseline --no-profile 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), round(d["value"],1))')"
done
TCQR_NN_PRE_ALL=0 H=512,256,128 python tools/gemm_bench.py; H=512,256,128 python tools/gemm_bench.py
