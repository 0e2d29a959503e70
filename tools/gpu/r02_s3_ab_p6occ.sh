# A/B: path 6 tile shrunk (<= 20 %) for one more Phase I CTA per SM at any
# occupancy below four (0x400000) vs only from one to two (the rule kept).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
for d in 0 0x400000 0 0x400000; do
  echo "dbg=$d"
  timeout 300 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 16,24,8 --kinds perm --variants p6 --runs "" --dbg $d
done > gpurun_out/s3/ab_p6occ.log 2>&1
cat gpurun_out/s3/ab_p6occ.log
