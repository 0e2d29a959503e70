# Session-3 check: smoke, default bench line, reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s3/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s3/smoke.log
timeout 1200 python bench.py > gpurun_out/s3/bench.json 2> gpurun_out/s3/bench.err; echo "bench rc=$?"
tail -c 400 gpurun_out/s3/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s3/ref.json 2> gpurun_out/s3/ref.err; echo "ref rc=$?"
tail -c 300 gpurun_out/s3/ref.json
