cd $GRAFT_REPO_ROOT
for kb in 8 4 2; do
  echo "TN_MINKB=$kb: $(TCQR_TN_MINKB=$kb timeout 300 python bench.py --steps 5 --warmup 3 --no-lls --no-e2e --no-configs --no-cpu-baseline --no-profile 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), round(d["value"],1))')"
done
