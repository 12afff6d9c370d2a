# Round-2 evidence at HEAD: full ncu capture of one whole-leaf launch, the bench's launch list
# (cold-cache, serialized per-launch times), and the tensor-pipe / DRAM captures of ncu_evidence.sh.
cd $GRAFT_REPO_ROOT
bash tools/gpu/ncu_leaf.sh
python tools/ncu_summary.py gpurun_out/leaf_full.ncu-rep > gpurun_out/ncu_leaf_summary.txt 2>&1
ncu -i gpurun_out/leaf_full.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__warp_issue_stalled_barrier_per_warp_active.pct,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/ncu_leaf_raw.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2200 --csv --log-file gpurun_out/launches_v2.csv python bench.py --steps 2 --warmup 1 --no-lls --no-e2e --no-configs --no-cpu-baseline --no-profile > gpurun_out/ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/launches_v2.csv > gpurun_out/launches_v2_summary.txt 2>&1
bash tools/gpu/ncu_evidence.sh > /dev/null 2>&1
cat gpurun_out/ncu_leaf_summary.txt gpurun_out/launches_v2_summary.txt | head -60
