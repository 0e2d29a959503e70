cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_seq3.py -x -q 2>&1 | tail -1
for n in 16777216 67108864; do
timeout 900 python scratch/ab_chain/tools/skew_probe.py --n-src $n --n-out $n --recs 8,12,16,24,32 --kinds perm --runs "" --variants "" --reps 3 | sed "s/^/OLD $n /"
timeout 900 python tools/skew_probe.py --n-src $n --n-out $n --recs 8,12,16,24,32 --kinds perm --runs "" --variants "" --reps 3 | sed "s/^/NEW $n /"
done
timeout 900 python scratch/ab_chain/tools/skew_probe.py --n-src 134217728 --n-out 134217728 --recs 8,16 --kinds perm --runs "" --variants "" --reps 3 | sed "s/^/OLD 2^27 /"
timeout 900 python tools/skew_probe.py --n-src 134217728 --n-out 134217728 --recs 8,16 --kinds perm --runs "" --variants "" --reps 3 | sed "s/^/NEW 2^27 /"
