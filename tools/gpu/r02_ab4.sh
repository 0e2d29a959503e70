cd $GRAFT_REPO_ROOT
for d in 0 500 1000 2000 4000; do
DPG_P2_DBG=$d python tools/skew_probe.py --recs 256 --kinds uniform,exp --runs "" --variants p2 | sed "s/^/DBG $d /"
DPG_P2_DBG=$d python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 256,128 --kinds perm --runs "" --variants p2 | sed "s/^/DBG $d /"
done
