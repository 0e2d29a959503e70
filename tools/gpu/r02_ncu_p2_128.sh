cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/p2b
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe_gather -s 1 -c 1 \
    -o gpurun_out/p2b/probe128 python tools/one_seq3.py --rec 128 --path 2 > gpurun_out/p2b/ncu.log 2>&1
echo "ncu rc=$?"
