# Session-3 verification after a planner change: GPU tests and the bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3/gputest2.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/s3/gputest2.log
timeout 1200 python bench.py > gpurun_out/s3/bench2.json 2> gpurun_out/s3/bench2.err; echo "bench rc=$?"
