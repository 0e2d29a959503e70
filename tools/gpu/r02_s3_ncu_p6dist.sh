# ncu of path 6's Phase I (k3_distribute) on 16 Mi x 4 B after the occupancy rule.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
timeout 300 python tools/one_seq3.py --rec 4 --path 6 > gpurun_out/s3/one4.log 2>&1; echo "one rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k3_" -c 6 \
    -o gpurun_out/s3/ncu_p6_rec4 python tools/one_seq3.py --rec 4 --path 6 > gpurun_out/s3/ncu4.log 2>&1
echo "ncu rc=$?"
