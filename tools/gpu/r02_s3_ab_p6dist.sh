# A/B: path 6 Phase I occupancy for 4-byte records (one 117 KB Phase I CTA per SM):
# 0x200000 = 1024 threads per CTA, 0x400000 = tile shrunk so that two CTAs fit an SM.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
for d in 0 0x200000 0x400000 0 0x200000 0x400000; do
  echo "dbg=$d"
  timeout 300 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 4,8 --kinds perm --variants p6 --runs "" --dbg $d
  timeout 300 python tools/skew_probe.py --n-src 67108864 --n-out 67108864 --recs 4 --kinds perm --variants p6 --runs "" --dbg $d
done > gpurun_out/s3/ab_p6dist.log 2>&1
cat gpurun_out/s3/ab_p6dist.log
