# ncu of path 2 with radix Phase I on c3a 256 B (16 Mi permutation), and the
# 64 B case with both Phase I variants timed.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/radix
timeout 300 python tools/one_seq3.py --rec 256 --path 2 > gpurun_out/radix/one.log 2>&1; echo "one rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sort_pass|k_run_bounds|k_probe_gather|k_item" -c 12 \
    -o gpurun_out/radix/ncu_c3a256_p2 python tools/one_seq3.py --rec 256 --path 2 > gpurun_out/radix/ncu.log 2>&1
echo "ncu rc=$?"
timeout 900 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 64,100,128,256 --kinds perm --variants p1,p2,p2r,p5 --runs "" > gpurun_out/radix/probe.log 2>&1
echo "probe rc=$?"; cat gpurun_out/radix/probe.log
