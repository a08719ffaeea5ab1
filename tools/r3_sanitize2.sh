cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck; do
  for t in "bert 32" "vgg16 16" "mobilenet_v2 64"; do
    f=gpurun_out/sanitize/${tool}_$(echo $t | tr ' ' '_').log
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py $t > $f 2>&1
    echo "$tool $t rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $f | tail -1)"
  done
done
