cd $GRAFT_REPO_ROOT
for ic in 0 1; do B2_IM2COL=$ic timeout 60 python tools/conv_micro.py 256 224 224 8 64 7 2; done
B2_IM2COL=1 timeout 60 python tools/conv_micro.py 256 224 224 8 32 3 2
DTS=1 timeout 300 python tools/gpu_check.py resnet50,mobilenet_v2 2>&1 | tail -6
timeout 120 python tools/profile_ops.py resnet50 256 1 > gpurun_out/prof_r50.txt 2>&1
