# Skew partitions (section 2.3): GPU parity tests, then the plan comparison.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_skew.py -x -q > gpurun_out/skew_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/skew_tests.log
tail -30 gpurun_out/skew_tests.log
timeout 900 python tools/skew_probe.py > gpurun_out/skew_probe.log 2>&1; echo "probe rc=$?"
cat gpurun_out/skew_probe.log
