cd $GRAFT_REPO_ROOT
timeout 1500 python tools/skew_probe.py --n-src 67108864 --n-out 67108864 --recs 48,64,100 --kinds perm --runs "" --variants p2,p5 --reps 3
timeout 900 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 12,24,32 --kinds perm --runs "" --variants p1,p1g2,p2 --reps 5
