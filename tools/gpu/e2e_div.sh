cd $GRAFT_REPO_ROOT
for d in 8 16 32 64; do
  echo "div=$d: $(TCQR_STREAM_DIV=$d timeout 300 python bench.py --steps 3 --warmup 3 --no-lls --no-configs --no-cpu-baseline --no-profile 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["e2e"]["ms_per_step"],2))')"
done
