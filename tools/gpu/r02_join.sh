cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "join or skew or fk" 2>&1 | tail -3
timeout 900 python bench.py --config c4 --steps 5 --warmup 2 --no-cpu > gpurun_out/join_c4.json 2>&1
python - <<'PY'
import json
d=json.loads(open('gpurun_out/join_c4.json').read().strip().splitlines()[-1])
print('dpg', d['ms'], d['config'], d['phases_ms'])
for k in ('direct','dpg_seq3','dpg_sort_join'): print(k, d[k]['ms'], d[k].get('plan_path'))
PY
