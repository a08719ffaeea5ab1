cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "" "B2_DEV=1 B2_PAIR=0 B2_SPLIT=0" "B2_DEV=1 B2_PAIR=0" "B2_DEV=1 B2_PAIR=0 B2_SPLIT=0 B2_CHAIN=0" "B2_DEV=1 B2_PAIR=0 B2_SPLIT=0 B2_BAND=0"; do
  env $cfg timeout 300 python tools/det_layers.py resnet50 256 4 >> gpurun_out/det.log 2>&1
  env $cfg B2_LIB=ab/libb2_base.so timeout 300 python tools/det_layers.py resnet50 256 4 | sed 's/^/BASE /' >> gpurun_out/det.log 2>&1
done
cat gpurun_out/det.log
