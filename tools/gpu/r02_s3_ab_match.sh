# A/B: the radix Phase I rank by one match.any (dbg 0x100000) vs eight ballots.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
for d in 0 0x100000 0 0x100000; do
  echo "dbg=$d"
  timeout 600 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 128,256 --kinds perm --variants p2 --runs "" --dbg $d
  timeout 600 python tools/skew_probe.py --n-src 16777216 --n-out 67108864 --recs 256 --kinds uniform --variants p2 --runs "" --dbg $d
done > gpurun_out/s3/ab_match.log 2>&1
cat gpurun_out/s3/ab_match.log
