cd $GRAFT_REPO_ROOT
for m in "mlp 1" "mlp 16" "mlp 64" "mlp 256"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_base.so AB_LABEL=base timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
sort -k2,3 -s gpurun_out/ab.txt
timeout 1500 python -m pytest tests/test_gpu.py -q -rf -x -k "mlp or parity" 2>&1 | tail -3
