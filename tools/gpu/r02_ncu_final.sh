# ncu --set full of the round-2 kernels on their configurations: path 2 (radix
# Phase I with run boundaries, work items, probe-gather) on c3a 256 B; path 6
# on c3a 8 B; the c2 headline kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncuf
timeout 300 python tools/one_seq3.py --rec 256 --path 2 > /dev/null 2>&1; echo "one rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sort_pass|k_probe_gather|k_item" -s 5 -c 5 \
    -o gpurun_out/ncuf/c3a256_p2 python tools/one_seq3.py --rec 256 --path 2 > gpurun_out/ncuf/p2.log 2>&1; echo "p2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_ -s 4 -c 4 \
    -o gpurun_out/ncuf/c3a8_p6 python tools/one_seq3.py --rec 8 > gpurun_out/ncuf/p6.log 2>&1; echo "p6 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dpg_l2run -c 1 \
    -o gpurun_out/ncuf/c2_l2run python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extras > gpurun_out/ncuf/c2.log 2>&1; echo "c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/ncuf/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncuf/launches.log 2>&1; echo "launches rc=$?"
