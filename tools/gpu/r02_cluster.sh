cd $GRAFT_REPO_ROOT
for cl in 1 2 4 8; do
  echo "== cluster $cl"
  DPG_SEQ3_CLUSTER=$cl timeout 300 python tools/seq3_probe.py --n 16777216 --recs 8,16,32 --kinds perm --reps 5 2>&1 | tail -3
  DPG_SEQ3_CLUSTER=$cl timeout 300 python tools/seq3_probe.py --n 67108864 --recs 8,16 --kinds perm --reps 3 2>&1 | tail -2
done
