# depthwise strip kernel: bf16 pair pack + packed ReLU6 — parity + A/B against HEAD
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_conv.py -q -rf -x 2>&1 | tail -2
for rep in 1 2 3; do
for m in "mobilenet_v2 256" "mobilenet_v2 16"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_dw.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_dw.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab_dw.txt | grep -v "^ \|Trace\|File"
