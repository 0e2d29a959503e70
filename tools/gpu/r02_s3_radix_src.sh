# Session-3 sanity + source-level ncu of path 2's radix Phase I passes (c3a 128 B,
# 16 Mi permutation) and their timing.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3/gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/s3/gputest.log
timeout 300 python tools/one_seq3.py --rec 128 --path 2 > gpurun_out/s3/one.log 2>&1; echo "one rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sort_pass" -c 2 \
    -o gpurun_out/s3/ncu_radix128 python tools/one_seq3.py --rec 128 --path 2 > gpurun_out/s3/ncu.log 2>&1
echo "ncu rc=$?"
timeout 600 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 128,256 --kinds perm --variants p2 --runs "" > gpurun_out/s3/probe.log 2>&1
echo "probe rc=$?"; cat gpurun_out/s3/probe.log
