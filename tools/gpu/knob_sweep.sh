# in-place sweep of tuning switches (config 3 factor time from tools/leaf_gaps.py), interleaved
cd $GRAFT_REPO_ROOT
f() { env "$@" python tools/leaf_gaps.py 2>&1 | tail -8 | head -1 | cut -c1-16; }
echo "warmup $(f X=1)"
for r in 1 2 3; do
  echo "LA_W=1024 $(f TCQR_LOOKAHEAD_W=1024)"
  echo "default $(f X=1)"
  echo "LA_W=1024+RES0 $(f TCQR_LOOKAHEAD_W=1024 TCQR_LEAF_RESERVE=0)"
  echo "RESERVE=0 $(f TCQR_LEAF_RESERVE=0)"
  echo "MINKB=16 $(f TCQR_TN_MINKB=16)"
done
