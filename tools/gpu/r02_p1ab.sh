cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 300 python scratch/ab_chain/tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 64,100 --kinds perm --runs "" --variants p1 | sed "s/^/OLD /"
timeout 300 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 64,100 --kinds perm --runs "" --variants p1 | sed "s/^/NEW /"
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -x -q -k "forced or guard or sweep" 2>&1 | tail -1
