cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for part in leaf panel proj gemm cgls vranks; do
    echo "== $tool $part"
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py $part 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|========= (Invalid|Race|Barrier|Error|Warning)|sanitize_run|Traceback|Error" | head -12
  done
done > gpurun_out/sanitize.txt 2>&1
cat gpurun_out/sanitize.txt
