cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/gputests.log 2>&1
tail -4 gpurun_out/gputests.log
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu.py -q -rf -k "determinism" 2>&1 | tail -1 >> gpurun_out/det_rep.log; done
cat gpurun_out/det_rep.log
for m in "resnet50 256" "bert 128" "vgg16 256" "mobilenet_v2 256" "resnet50 16"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab4.log 2>&1
done
cat gpurun_out/ab4.log
