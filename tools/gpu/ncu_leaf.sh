cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:leaf_kernel -s 2 -c 1 \
  -o gpurun_out/leaf_full python tools/leaf_one.py 32768 > gpurun_out/ncu_leaf.log 2>&1
tail -3 gpurun_out/ncu_leaf.log
