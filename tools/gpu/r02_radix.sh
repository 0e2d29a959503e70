# Radix Phase I for path 2: parity, then the skew probe and c3a256 phases.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_skew.py -x -q -k "not slow" > gpurun_out/radix_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/radix_tests.log
tail -25 gpurun_out/radix_tests.log
timeout 900 python tools/skew_probe.py --recs 64,256 --runs 1024 > gpurun_out/skew_probe3.log 2>&1; echo "probe rc=$?"
cat gpurun_out/skew_probe3.log
