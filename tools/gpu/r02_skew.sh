# Skew partitions (section 2.3): the plan comparison on skewed rid lists.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/skew_probe.py "$@" > gpurun_out/skew_probe.log 2>&1; echo "probe rc=$?"
cat gpurun_out/skew_probe.log
