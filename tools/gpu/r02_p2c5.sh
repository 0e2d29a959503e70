cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_skew.py tests/test_gpu_parity.py -x -q -k "not slow" 2>&1 | tail -2
timeout 900 python tools/skew_probe.py --n-src 134217728 --n-out 67108864 --recs 100 --kinds uniform --runs "" --variants p2,p5 --reps 3
timeout 900 python bench.py --config c4x --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4x', d['value'], d['ms_per_step'], d['config'].get('plan_path'))"
