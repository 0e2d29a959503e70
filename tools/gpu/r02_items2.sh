cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_skew.py tests/test_gpu_parity.py -x -q -k "not slow" 2>&1 | tail -2
for i in 1 2; do
python scratch/ab_old/tools/skew_probe_new.py --n-src 16777216 --n-out 16777216 --recs 256,128,64 --kinds perm --variants p2 --runs "" --reps 7 | sed "s/^/OLD /"
python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 256,128,64 --kinds perm --variants p2,p2g --runs "" --reps 7 | sed "s/^/NEW /"
done
python tools/skew_probe.py --recs 64,256 --runs 1024 --variants p2,p5
