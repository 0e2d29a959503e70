cd $GRAFT_REPO_ROOT
timeout 2000 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scratch/ab_chain/tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 40,48,72,96,100,120 --kinds perm --runs "" --variants p1 | sed "s/^/OLD /"
timeout 300 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 40,48,72,96,100,120 --kinds perm --runs "" --variants p1 | sed "s/^/NEW /"
