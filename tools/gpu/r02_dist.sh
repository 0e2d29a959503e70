cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "invalid_fk or two_host or segments" 2>&1 | tail -3
