# Session-3 baseline: whole GPU suite, bench, per-op profiles of ResNet-50 and BERT
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
for m in "resnet50 256" "bert 128" "vgg16 256" "mobilenet_v2 256" "resnet50 16" "resnet50 1"; do
  timeout 300 python tools/fwd_time.py $m >> gpurun_out/fwd.txt 2>&1
done
timeout 300 python tools/profile_ops.py bert 128 0 > gpurun_out/ops_bert.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/gputests.log 2>&1
tail -3 gpurun_out/gputests.log; cat gpurun_out/fwd.txt
