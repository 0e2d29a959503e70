cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_skew.py tests/test_gpu_guard.py -x -q -k "radix or histogram or skew or forced or guard or config_3 or bounds or segments or sweep" 2>&1 | tail -1
for i in 1 2; do
timeout 300 python scratch/ab_chain/tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 64,128,256 --kinds perm --runs "" --variants p2 | sed "s/^/OLD /"
timeout 300 python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 64,128,256 --kinds perm --runs "" --variants p2 | sed "s/^/NEW /"
done
timeout 300 python scratch/ab_chain/tools/skew_probe.py --recs 256,64 --kinds uniform,exp --runs "" --variants p2 | sed "s/^/OLD /"
timeout 300 python tools/skew_probe.py --recs 256,64 --kinds uniform,exp --runs "" --variants p2 | sed "s/^/NEW /"
