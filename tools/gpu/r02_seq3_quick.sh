cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_seq3.py -x -q 2>&1 | tail -2
timeout 600 python tools/seq3_probe.py --recs 8,16,32 --kinds perm,repl 2>&1 | tail -6
timeout 300 python tools/seq3_phase2_exp.py 2>&1 | tail -12
