cd $GRAFT_REPO_ROOT
for o in 1 2; do
DPG_RADIX_OCC=$o timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "radix or histogram" 2>&1 | tail -1
DPG_RADIX_OCC=$o python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 128,256 --kinds perm --runs "" --variants p2 | sed "s/^/OCC $o /"
DPG_RADIX_OCC=$o python tools/skew_probe.py --recs 256 --kinds uniform,zipf --runs "" --variants p2 | sed "s/^/OCC $o /"
done
