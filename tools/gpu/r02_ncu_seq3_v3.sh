cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_seq3.py -x -q 2>&1 | tail -3
timeout 600 python tools/seq3_probe.py --recs 8,16,32 --kinds perm 2>&1 | tail -5
python tools/one_seq3.py --rec 8 && \
ncu --set full --clock-control none --import-source on -k regex:k3_ -c 4 -o gpurun_out/ncu_seq3v3_r8 python tools/one_seq3.py --rec 8 > gpurun_out/ncu_full3.log 2>&1
tail -1 gpurun_out/ncu_full3.log
