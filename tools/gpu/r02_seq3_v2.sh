cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_seq3.py -x -q 2>&1 | tail -15
timeout 600 python tools/seq3_probe.py --recs 4,8,16,32,64 --kinds perm 2>&1 | tail -20
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "forced_path" 2>&1 | tail -3
