cd $GRAFT_REPO_ROOT
for cl in 1 2 4; do
  echo "== cluster $cl"
  DPG_SEQ3_CLUSTER=$cl timeout 300 python tools/seq3_probe.py --n 134217728 --recs 8 --kinds perm --reps 3 2>&1 | tail -1
done
