cd $GRAFT_REPO_ROOT
bash tools/gpu/sanitize.sh > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/gpu_suite.log
grep -E "SUMMARY|Error:" gpurun_out/sanitize.txt | sort | uniq -c; tail -3 gpurun_out/gpu_suite.log
