# deep-level probes: leaf gaps (default and without look-ahead), ncu of the TN / NN at h = 512, 1024
cd $GRAFT_REPO_ROOT
python tools/leaf_gaps.py 2>&1 | tail -8
echo "== TCQR_LOOKAHEAD_W=0"; TCQR_LOOKAHEAD_W=0 python tools/leaf_gaps.py 2>&1 | tail -8
N="ncu --set full --import-source on --clock-control none"
for H in 128 512 1024; do
  H=$H timeout 600 $N -k regex:"tc_gemm|finalize|splitk" -s 3 -c 3 -o gpurun_out/ncu_gemm_h$H python tools/gemm_one.py > gpurun_out/ncu_gemm_h$H.log 2>&1
  echo "== H=$H"; python tools/ncu_summary.py gpurun_out/ncu_gemm_h$H.ncu-rep 2>&1 | cut -c1-400
done
