cd $GRAFT_REPO_ROOT
python tools/one_seq3.py --rec 8 && \
ncu --set full --clock-control none --import-source on -k regex:k3_ -c 4 -o gpurun_out/ncu_seq3v2_r8 python tools/one_seq3.py --rec 8 > gpurun_out/ncu_full2.log 2>&1
tail -3 gpurun_out/ncu_full2.log
