# ncu --set full + source of single launches of one ResNet-50 b=256 forward:
# layer3 expand (tc_gemm2 #7), layer1 block-0 chain (#1), layer2 block-0 chain (#4), layer2 3x3 band (#1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cap() {  # name regex skip
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$2 --launch-skip $3 --launch-count 1 \
    -o gpurun_out/r3_$1 python tools/ncu_target.py resnet50 256 > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
}
cap expand tc_gemm2_kernel 6
cap chain1 chain_gemm_kernel 0
cap chain4 chain_gemm_kernel 3
cap band128 "conv_band_kernel" 0
ls -la gpurun_out/*.ncu-rep
