cd $GRAFT_REPO_ROOT
for i in 1 2; do
(cd scratch/ab_old && timeout 300 python bench.py --config c4 --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('OLD c4', round(d['ms'],3), 'sortjoin', round(d['dpg_sort_join']['ms'],3), 'seq3', round(d['dpg_seq3']['ms'],3))")
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('NEW c4', round(d['ms'],3), 'sortjoin', round(d['dpg_sort_join']['ms'],3), 'seq3', round(d['dpg_seq3']['ms'],3))"
done
