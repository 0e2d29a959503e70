cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_skew.py tests/test_gpu_parity.py -x -q -k "not slow" 2>&1 | tail -2
python tools/skew_probe.py --recs 256,64 --kinds uniform,exp,zipf,hot --runs "" --variants p2,p5
python tools/skew_probe.py --n-src 16777216 --n-out 16777216 --recs 256,128,64 --kinds perm --runs "" --variants p1,p2
python scratch/ab_chain/tools/skew_probe_new.py --recs 256,64 --kinds uniform,exp,zipf --runs "" --variants p2 | sed "s/^/CHAIN /"
