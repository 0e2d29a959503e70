# ncu of the path-6 kernels (c3 shape, rec 8 and 32): launch list + one full capture each
cd $GRAFT_REPO_ROOT
python tools/one_seq3.py --rec 8 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests.sum,lts__t_sectors.sum --clock-control none --csv \
    python tools/one_seq3.py --rec 8 > gpurun_out/ncu_seq3_r8_metrics.csv 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests.sum,lts__t_sectors.sum --clock-control none --csv \
    python tools/one_seq3.py --rec 32 > gpurun_out/ncu_seq3_r32_metrics.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:k3_ -c 6 -o gpurun_out/ncu_seq3_r8 python tools/one_seq3.py --rec 8 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
