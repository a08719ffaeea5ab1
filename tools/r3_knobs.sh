# A/B of existing dev knobs on ResNet-50 b=256 / BERT b=128 after this round's kernel changes
cd $GRAFT_REPO_ROOT
for cfg in "" "B2_FOLD_MAX_K=0" "B2_FOLD_MAX_K=256" "B2_ALT_ORDER=0" "B2_PAIR_MIN_K=512" "B2_BAND_PAIR=0"; do
  env B2_DEV=1 $cfg AB_LABEL="${cfg:-default}" timeout 300 python tools/fwd_time.py resnet50 256 >> gpurun_out/knobs.txt 2>&1
done
for cfg in "" "B2_FOLD_MAX_K=0" "B2_ALT_ORDER=0"; do
  env B2_DEV=1 $cfg AB_LABEL="${cfg:-default}" timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/knobs.txt 2>&1
done
for cfg in "" "B2_FOLD_MAX_K=0"; do
  env B2_DEV=1 $cfg AB_LABEL="${cfg:-default}" timeout 300 python tools/fwd_time.py mobilenet_v2 256 >> gpurun_out/knobs.txt 2>&1
done
cat gpurun_out/knobs.txt
