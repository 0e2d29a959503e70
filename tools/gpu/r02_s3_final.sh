# Session-3 final: the new path 6 tests, compute-sanitizer on the small calls, full GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
timeout 600 python -m pytest tests/test_gpu_seq3.py -q -x -k shrunk > gpurun_out/s3/shrunk.log 2>&1; echo "shrunk rc=$?"; tail -2 gpurun_out/s3/shrunk.log
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/s3/san_$t.log 2>&1; echo "$t rc=$?"; tail -2 gpurun_out/s3/san_$t.log
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3/gputest3.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/s3/gputest3.log
