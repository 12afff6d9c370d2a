cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qr_lls.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "lls or solve or gemv" > gpurun_out/lls_tests.log 2>&1
echo "rc=$?" >> gpurun_out/lls_tests.log
timeout 600 env REORTH=0 python tools/lls_bench.py > gpurun_out/lls_prof_paper.txt 2>&1
tail -2 gpurun_out/lls_tests.log; grep -v "^solve 0" gpurun_out/lls_prof_paper.txt | cut -c1-150
