cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seq3.py -x -q -k "join" 2>&1 | tail -1
for c in c4 c4x; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['config']['plan_path'], round(d['ms'],3), 'direct', round(d['direct']['ms'],3), 'seq3', round(d['dpg_seq3']['ms'],3), 'sortjoin', round(d['dpg_sort_join']['ms'],3), 'ok', d['parity_sampled_ok'])"
done
