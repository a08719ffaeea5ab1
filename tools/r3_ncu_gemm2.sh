cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tc_gemm2_kernel --launch-skip 28 --launch-count 28 \
    -o gpurun_out/r3_gemm2_all python tools/ncu_target.py resnet50 256 > gpurun_out/ncu_gemm2_all.log 2>&1
echo rc=$?; ls -la gpurun_out/r3_gemm2_all.ncu-rep
