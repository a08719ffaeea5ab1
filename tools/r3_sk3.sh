cd $GRAFT_REPO_ROOT
export B2_DEV=1
B2_SK=0 timeout 120 python tools/conv_micro.py 256 14 14 1024 256 1 1 2>&1 | tail -1
B2_SK=3 timeout 120 python tools/conv_micro.py 256 14 14 1024 256 1 1 2>&1 | tail -1
B2_SK=2 timeout 120 python tools/conv_micro.py 256 14 14 1024 256 1 1 2>&1 | tail -1
B2_SK=0 timeout 120 python tools/gemm_micro.py 16384 3072 768 res 2>&1 | tail -1
B2_SK=1 timeout 120 python tools/gemm_micro.py 16384 3072 768 res 2>&1 | tail -1
B2_SK=0 timeout 120 python tools/gemm_micro.py 16384 768 768 res 2>&1 | tail -1
B2_SK=1 timeout 120 python tools/gemm_micro.py 16384 768 768 res 2>&1 | tail -1
