# Final checks: smoke(), the reference arm, the bench line, GPU tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final/smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final/ref.json 2> gpurun_out/final/ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/final/ref.json
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/final/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final/gputest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench rc=$?"
