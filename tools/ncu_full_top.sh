# ncu --set full of the top kernels of one ResNet-50 b=256 forward (first launch of each)
cd $GRAFT_REPO_ROOT
for k in chain_gemm_kernel tc_gemm2_kernel tc_gemm_kernel conv_band_pair_kernel conv_band_kernel stem_pool_kernel; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/full_$k python tools/profile_ops.py resnet50 256 > /dev/null 2>&1
done
