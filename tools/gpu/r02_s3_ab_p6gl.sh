# A/B: path 6 Phase I with the rids read from global memory twice (0x800000, no
# shared-memory rid stage: 2-4 CTAs per SM) against the staged tile.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
for d in 0 0x800000 0 0x800000; do
  echo "dbg=$d"
  timeout 300 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 4,8,16 --kinds perm --variants p6 --runs "" --dbg $d
  timeout 300 python tools/skew_probe.py --n-src 67108864 --n-out 67108864 --recs 4,8,16 --kinds perm --variants p6 --runs "" --dbg $d
  timeout 300 python tools/skew_probe.py --n-src 134217728 --n-out 134217728 --recs 8 --kinds perm --variants p6 --runs "" --dbg $d
done > gpurun_out/s3/ab_p6gl.log 2>&1
cat gpurun_out/s3/ab_p6gl.log
