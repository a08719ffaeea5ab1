cd $GRAFT_REPO_ROOT
for sd in 0 1; do B2_S2D=$sd timeout 60 python tools/conv_micro.py 256 224 224 3 64 7 2; done
for sd in 0 1; do B2_S2D=$sd timeout 60 python tools/conv_micro.py 256 224 224 3 32 3 2; done
DTS=1 timeout 300 python tools/gpu_check.py resnet50,mobilenet_v2 2>&1 | tail -6
timeout 120 python tools/profile_ops.py resnet50 256 1 > gpurun_out/prof_r50.txt 2>&1
timeout 120 python tools/profile_ops.py mobilenet_v2 256 1 > gpurun_out/prof_mnv2.txt 2>&1
