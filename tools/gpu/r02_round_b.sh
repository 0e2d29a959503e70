# Round-2 evidence, second pass: GPU tests, the bench line (with c3a128 and
# c4x nested), the skew comparison, and an ncu launch list of the bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof2
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/prof2/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/prof2/gputest.log
tail -3 gpurun_out/prof2/gputest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/prof2/bench.json 2> gpurun_out/prof2/bench.err
echo "bench rc=$?"
timeout 1200 python tools/skew_probe.py --recs 64,256 --kinds exp,hot,zipf,uniform --runs 1024 --variants p1,p2,p5 > gpurun_out/prof2/skew.log 2>&1
echo "skew rc=$?"
timeout 900 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 64,128,256 --kinds perm --runs "" --variants p1,p2,p2g > gpurun_out/prof2/p2perm.log 2>&1
echo "p2perm rc=$?"
