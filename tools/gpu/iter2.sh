cd $GRAFT_REPO_ROOT

timeout 300 python tools/leaf_phases.py 32768 > gpurun_out/leaf_phases.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_qr_lls.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/leaf_tests.log 2>&1
echo "rc=$?" >> gpurun_out/leaf_tests.log
timeout 600 python -m pytest tests/test_gpu_vranks.py -x -q -p no:cacheprovider > gpurun_out/vranks.log 2>&1
echo "rc=$?" >> gpurun_out/vranks.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -2 gpurun_out/leaf_tests.log gpurun_out/vranks.log; head -4 gpurun_out/leaf_phases.txt; cut -c1-200 gpurun_out/bench_quick.json
