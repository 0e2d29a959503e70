cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe_gather -s 1 -c 1 \
    -o gpurun_out/ab/chain64 python scratch/ab_chain/tools/one_p2.py > gpurun_out/ab/c.log 2>&1
echo "chain rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe_gather -s 1 -c 1 \
    -o gpurun_out/ab/uint64 python tools/one_p2.py > gpurun_out/ab/u.log 2>&1
echo "uint4 rc=$?"
