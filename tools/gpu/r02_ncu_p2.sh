# ncu --set full of path 2 (radix Phase I passes, run bounds, work items,
# probe-gather) on c3a 256 B (16 Mi permutation).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/p2
timeout 300 python tools/one_seq3.py --rec 256 --path 2 > gpurun_out/p2/one.log 2>&1; echo "one rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sort_pass|k_run_bounds|k_probe_gather|k_item" -s 6 -c 6 \
    -o gpurun_out/p2/ncu_c3a256_p2 python tools/one_seq3.py --rec 256 --path 2 > gpurun_out/p2/ncu.log 2>&1
echo "ncu rc=$?"
