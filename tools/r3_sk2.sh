# split-tail micro: one 1x1 conv with 196 pair tiles, B2_SK off / auto / forced
cd $GRAFT_REPO_ROOT
for v in 0 1 2 3; do
  echo "B2_SK=$v"; B2_SK=$v timeout 120 python tools/conv_micro.py 256 14 14 1024 256 1 1 2>&1 | tail -1
done
B2_SK=0 timeout 120 python tools/gemm_micro.py 16384 3072 768 res 2>&1 | tail -1
B2_SK=1 timeout 120 python tools/gemm_micro.py 16384 3072 768 res 2>&1 | tail -1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm2 -c 1 -o gpurun_out/sk3 python tools/conv_micro.py 256 14 14 1024 256 1 1 > /dev/null 2>&1
ls -la gpurun_out/sk3.ncu-rep
