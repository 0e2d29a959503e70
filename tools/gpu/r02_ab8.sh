cd $GRAFT_REPO_ROOT
for d in 0x100000 0 0x80000; do
DPG_P2_DBG=$d python tools/skew_probe.py --recs 256,64 --kinds uniform,exp,zipf --runs "" --variants p2 | sed "s/^/DBG $d /"
DPG_P2_DBG=$d python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 256,128 --kinds perm --runs "" --variants p2 | sed "s/^/DBG $d /"
done
python scratch/ab_chain/tools/skew_probe_new.py --recs 256,64 --kinds uniform,exp,zipf --runs "" --variants p2 | sed "s/^/CHAIN /"
