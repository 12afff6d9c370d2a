# bench (config 3 only) under L2 hint masks, interleaved
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in 0 7 5 6; do
  echo "EF=$v $(TCQR_L2_EF=$v python bench.py --steps 10 --warmup 3 --no-lls --no-e2e --no-configs --no-cpu-baseline --no-profile 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],3))')"
done; done
