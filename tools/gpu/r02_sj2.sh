cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sj
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sj/old.csv python scratch/ab_old/tools/one_sortjoin.py > /dev/null 2>&1; echo "old rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sj/new.csv python tools/one_sortjoin.py > /dev/null 2>&1; echo "new rc=$?"
