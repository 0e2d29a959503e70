# DPG (automatic plan) against the direct gather over record sizes, at 16 Mi
# and 64 Mi records (permutations), for profiles/r02_sweep_final.md.
cd $GRAFT_REPO_ROOT
timeout 900 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 4,8,12,16,24,32,48,64,96,100,128,256 --kinds perm --runs "" --variants "" --reps 5
timeout 1500 python tools/skew_probe.py --n-src 67108864 --n-out 67108864 --recs 4,8,12,16,24,32,48,64,100,128,256 --kinds perm --runs "" --variants "" --reps 3
