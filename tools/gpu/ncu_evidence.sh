# ncu --set full captures for the roofline evidence of SURVEY 8(d): tensor-pipe % of the K3/K4
# tensor-core GEMMs at a top-level and a deep-level shape, DRAM % of the CGLS GEMVs and triangular
# applies, the tall-path panel kernel and the K1 cast.  One kernel per capture (ncu replays it).
cd $GRAFT_REPO_ROOT
N="ncu --set full --import-source on --clock-control none"
H=8192 timeout 600 $N -k regex:tc_gemm -s 2 -c 2 -o gpurun_out/ncu_gemm_top python tools/gemm_one.py > gpurun_out/ncu_gemm_top.log 2>&1
H=256 timeout 600 $N -k regex:tc_gemm -s 2 -c 2 -o gpurun_out/ncu_gemm_deep python tools/gemm_one.py > gpurun_out/ncu_gemm_deep.log 2>&1
REORTH=1 timeout 900 $N -k regex:"gemv_n_part|gemv_t_part|tri_n_part|tri_t_part" -s 40 -c 4 -o gpurun_out/ncu_cgls python tools/lls_bench.py > gpurun_out/ncu_cgls.log 2>&1
timeout 600 $N -k regex:"panel_pipe|cast_" -s 20 -c 2 -o gpurun_out/ncu_tall python tools/tall_one.py > gpurun_out/ncu_tall.log 2>&1
for f in gpurun_out/ncu_gemm_top gpurun_out/ncu_gemm_deep gpurun_out/ncu_cgls gpurun_out/ncu_tall; do
  echo "== $f"; python tools/ncu_summary.py $f.ncu-rep 2>&1 | cut -c1-400
done > gpurun_out/ncu_evidence.txt
cat gpurun_out/ncu_evidence.txt
