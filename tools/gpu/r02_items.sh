# Path 2 work items: parity (path-2 sweeps, skew tests), then the skew probe.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_skew.py tests/test_gpu_parity.py -x -q -k "not slow" > gpurun_out/items_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/items_tests.log
tail -5 gpurun_out/items_tests.log
timeout 1200 python tools/skew_probe.py --recs 64,256 --runs 1024 > gpurun_out/skew_probe2.log 2>&1; echo "probe rc=$?"
cat gpurun_out/skew_probe2.log
