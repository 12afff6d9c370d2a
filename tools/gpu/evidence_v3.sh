# Round-2 evidence at HEAD (v3): the default bench line, leaf gaps and in-situ leaf phases, the
# bench's ncu launch list and a full ncu capture of one whole-leaf launch.
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench_v5.json 2> gpurun_out/bench_v5.err
python tools/leaf_gaps.py > gpurun_out/leaf_gaps_v1.txt 2>&1
python tools/leaf_phases_insitu.py > gpurun_out/leaf_phases_insitu_v1.txt 2>&1
bash tools/gpu/ncu_leaf.sh
python tools/ncu_summary.py gpurun_out/leaf_full.ncu-rep > gpurun_out/ncu_leaf_summary.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2200 --csv --log-file gpurun_out/launches_v3.csv python bench.py --steps 2 --warmup 1 --no-lls --no-e2e --no-configs --no-cpu-baseline --no-profile > gpurun_out/ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/launches_v3.csv > gpurun_out/launches_v3_summary.txt 2>&1
tail -c 3000 gpurun_out/bench_v5.json; head -3 gpurun_out/leaf_gaps_v1.txt; cat gpurun_out/ncu_leaf_summary.txt | head -5; head -12 gpurun_out/launches_v3_summary.txt
