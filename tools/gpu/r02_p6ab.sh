cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 300 python scratch/ab_chain/tools/seq3_probe.py --recs 8,16 --kinds perm --reps 5 | sed "s/^/OLD /"
timeout 300 python tools/seq3_probe.py --recs 8,16 --kinds perm --reps 5 | sed "s/^/NEW /"
timeout 300 python scratch/ab_chain/tools/seq3_probe.py --n 67108864 --recs 8,16 --kinds perm --reps 3 | sed "s/^/OLD /"
timeout 300 python tools/seq3_probe.py --n 67108864 --recs 8,16 --kinds perm --reps 3 | sed "s/^/NEW /"
done
