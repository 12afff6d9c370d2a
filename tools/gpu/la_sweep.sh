cd $GRAFT_REPO_ROOT
for w in 512 1024 2048 4096; do
  for s in 10 20; do
    echo "LA_W=$w LA_SMS=$s: $(TCQR_LOOKAHEAD_W=$w TCQR_LA_SMS=$s timeout 300 python bench.py --steps 5 --warmup 3 --no-lls --no-e2e --no-configs --no-cpu-baseline --no-profile 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), round(d["value"],1))')"
  done
done
