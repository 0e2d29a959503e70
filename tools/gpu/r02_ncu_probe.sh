cd $GRAFT_REPO_ROOT
python tools/one_seq3.py --rec 8 && \
ncu --set full --clock-control none --import-source on -k regex:k3_probe -c 1 -o gpurun_out/ncu_probe_r8 python tools/one_seq3.py --rec 8 > gpurun_out/ncu_probe.log 2>&1
tail -1 gpurun_out/ncu_probe.log
