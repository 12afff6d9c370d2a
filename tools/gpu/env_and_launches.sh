cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_env_variants.py -q -p no:cacheprovider > gpurun_out/env_variants.log 2>&1
echo "rc=$?" >> gpurun_out/env_variants.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-lls --no-e2e --no-configs --no-cpu-baseline --no-profile > gpurun_out/launches_bench.log 2>&1
python tools/level_breakdown.py gpurun_out/launches_cfg3.csv 1 > gpurun_out/levels_cfg3.txt 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg3.csv > gpurun_out/launch_summary.txt 2>&1
tail -3 gpurun_out/env_variants.log; cat gpurun_out/levels_cfg3.txt; head -30 gpurun_out/launch_summary.txt
