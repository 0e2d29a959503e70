cd $GRAFT_REPO_ROOT
timeout 300 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 32,64,100 --kinds perm --runs "" --variants p1,p2,p2r
timeout 300 python tools/skew_probe.py --recs 64 --kinds uniform,exp --runs "" --variants p1,p2,p2r
timeout 300 python tools/skew_probe.py --n-src 1048576 --n-out 1048576 --recs 100 --kinds perm --runs "" --variants p2,p2r
