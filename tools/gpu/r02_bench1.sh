cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo "rc=$?"
tail -5 gpurun_out/bench1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench1_ref.json 2>&1
echo "rc=$?"
