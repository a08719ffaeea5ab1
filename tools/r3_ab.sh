# A/B of a knob over graph-replayed forwards + parity of the default path.
# usage: AB_KNOB="B2_RES_TMA=0" bash tools/r3_ab.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in ${AB_MODELS:-"resnet50 256" "bert 128" "vgg16 256" "mobilenet_v2 256" "resnet50 16"}; do
  AB_LABEL=default timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  env B2_DEV=1 $AB_KNOB AB_LABEL="$AB_KNOB" timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
cat gpurun_out/ab.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu.py -x -q 2>&1 | tail -5
