# Round-2 evidence: GPU tests, the bench line, its ncu launch list, ncu --set full
# captures of the headline kernel (c2: k_dpg_l2run) and of the path-6 kernels (c3a, 8 B).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/prof/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/prof/gputest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/prof/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/prof/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dpg_l2run -c 1 \
    -o gpurun_out/prof/ncu_c2_l2run python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extras \
    > gpurun_out/prof/ncu_c2.log 2>&1
echo "ncu c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_ -c 4 \
    -o gpurun_out/prof/ncu_c3a8_seq3 python tools/one_seq3.py --rec 8 > gpurun_out/prof/ncu_seq3.log 2>&1
echo "ncu seq3 rc=$?"
ls -la gpurun_out/prof
