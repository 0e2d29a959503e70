cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_skew.py -x -q -k "sort or radix or histogram or skew or forced" 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', d['ms_per_step'], 'sort', d['dpg_sort']['ms_per_sort'], d['dpg_sort']['launches_per_sort'])"
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', d['ms'], 'sortjoin', d['dpg_sort_join']['ms'])"
