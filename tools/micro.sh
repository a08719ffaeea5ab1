cd $GRAFT_REPO_ROOT
timeout 60 python tools/gemm_micro.py 802816 64 256 res 2>&1 | sort | uniq -c | sort -rn | head -8
timeout 40 python tools/gemm_micro.py 65536 64 256 res 2>&1 | sort | uniq -c | sort -rn | head -5
