cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/p6big
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_probe -s 1 -c 1 \
    -o gpurun_out/p6big/probe8_n26 python tools/one_seq3.py --rec 8 --n 67108864 > gpurun_out/p6big/ncu.log 2>&1
echo "ncu rc=$?"
