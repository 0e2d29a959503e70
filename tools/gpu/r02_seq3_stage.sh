cd $GRAFT_REPO_ROOT
for kb in 128 64 32; do echo "stage $kb KB"; DPG_SEQ3_STAGE_KB=$kb timeout 600 python tools/seq3_probe.py --recs 8,16,32 --kinds perm 2>&1 | tail -3; done
