cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
python scratch/ab_chain/tools/skew_probe_new.py --recs 256 --kinds uniform,exp --runs "" --variants p2 | sed "s/^/CHAIN /"
python tools/skew_probe.py --recs 256 --kinds uniform,exp --runs "" --variants p2 | sed "s/^/UINT4 /"
python scratch/ab_old/tools/skew_probe_new.py --recs 256 --kinds uniform,exp --runs "" --variants p2 | sed "s/^/OLD   /"
done
