# ncu --set full of the single-CTA N = 128 band conv (ResNet-50 layer2 3x3 at b=256)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_band -c 1 -o gpurun_out/band128 python tools/conv_micro.py 256 28 28 128 128 3 1 > gpurun_out/band128.log 2>&1
tail -3 gpurun_out/band128.log
ls -la gpurun_out/band128.ncu-rep
