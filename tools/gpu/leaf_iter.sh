# leaf iteration: pipe micro-benchmark, leaf parity tests, phase timings, a quick bench line
cd $GRAFT_REPO_ROOT
./tools/micro/pipe_rates > gpurun_out/pipe_rates.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_qr_lls.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/leaf_tests.log 2>&1
echo "rc=$?" >> gpurun_out/leaf_tests.log
timeout 300 python tools/leaf_phases.py 32768 1024 > gpurun_out/leaf_phases.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -2 gpurun_out/leaf_tests.log; head -3 gpurun_out/leaf_phases.txt; cut -c1-300 gpurun_out/bench_quick.json
timeout 600 python -m pytest tests/test_gpu_vranks.py -x -q -p no:cacheprovider > gpurun_out/vranks.log 2>&1
echo "rc=$?" >> gpurun_out/vranks.log
tail -3 gpurun_out/vranks.log
