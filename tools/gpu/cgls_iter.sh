cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qr_lls.py -x -q -p no:cacheprovider -k "lls or solve" > gpurun_out/lls_tests.log 2>&1
echo "rc=$?" >> gpurun_out/lls_tests.log
timeout 300 env REORTH=1 python tools/lls_bench.py > gpurun_out/lls_prof_reorth.txt 2>&1
timeout 600 env REORTH=0 python tools/lls_bench.py > gpurun_out/lls_prof_paper.txt 2>&1
tail -2 gpurun_out/lls_tests.log; cat gpurun_out/lls_prof_reorth.txt gpurun_out/lls_prof_paper.txt | grep -v "^solve 0"
bash tools/gpu/ncu_evidence.sh
