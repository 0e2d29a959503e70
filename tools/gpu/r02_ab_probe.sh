cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe_gather -s 1 -c 1 \
    -o gpurun_out/ab/old python scratch/ab_old/tools/one_seq3.py --rec 256 --path 2 > gpurun_out/ab/old.log 2>&1
echo "old rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe_gather -s 1 -c 1 \
    -o gpurun_out/ab/new python tools/one_seq3.py --rec 256 --path 2 --hist-mode 2 > gpurun_out/ab/new.log 2>&1
echo "new rc=$?"
