cd $GRAFT_REPO_ROOT
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
echo "rc=$?"; tail -3 gpurun_out/bench2.err
