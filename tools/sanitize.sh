# compute-sanitizer over every kernel family at small shapes (memcheck, racecheck, synccheck).
# Kernel mix per target: resnet50 b=16 (stem_pool, band_pair, chain, tc_gemm, CTA-pair
# tc_gemm2, split-K), mobilenet_v2 b=8 (band stem, depthwise, narrow-K), vgg16 b=2 (band
# CGW=8, column segments, fused pools), bert b=2 (attention, LN, GELU), fp32 resnet50 b=2 (3xTF32).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck; do
  for t in "resnet50 16" "mobilenet_v2 8" "vgg16 2" "bert 2" "mlp 4" "resnet50 2 0"; do
    f=gpurun_out/sanitize/${tool}_$(echo $t | tr ' ' '_').log
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py $t > $f 2>&1
    echo "$tool $t rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $f | tail -1)"
  done
done
