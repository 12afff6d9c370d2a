cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests/test_gpu_vranks.py -x -q -p no:cacheprovider > gpurun_out/vranks.log 2>&1
echo "vranks rc=$?" >> gpurun_out/vranks.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_vranks.py > gpurun_out/gpu_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/gpu_suite.log
tail -3 gpurun_out/vranks.log gpurun_out/gpu_suite.log
