cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_seq3.py -x -q 2>&1 | tail -1
timeout 300 python tools/seq3_probe.py --recs 8,16,32 --kinds perm,repl --reps 5
timeout 300 python tools/seq3_probe.py --n 67108864 --recs 8,16 --kinds perm --reps 3
