cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sort" 2>&1 | tail -2
for i in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', d['ms_per_step'], 'sort', d['dpg_sort'])"
done
