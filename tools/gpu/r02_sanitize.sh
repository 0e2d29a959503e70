cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san/$tool.log
done
