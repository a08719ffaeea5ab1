cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bert_mask.py tests/test_gpu_daemon.py tests/test_gpu.py -q -rf -k "mask or daemon or foreign or controller or gen_input or parity" > gpurun_out/t4.log 2>&1
tail -5 gpurun_out/t4.log
bash tools/r2_ab1.sh
