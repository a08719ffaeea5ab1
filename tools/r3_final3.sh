# after the pooled-band change: full GPU suite + VGG sanitizer runs + VGG profile
cd $GRAFT_REPO_ROOT
E=gpurun_out/ev3; mkdir -p $E gpurun_out/sanitize
timeout 2400 python -m pytest tests -m gpu -q -rf > $E/gputests.log 2>&1; tail -2 $E/gputests.log
for tool in memcheck racecheck synccheck; do
  for t in "vgg16 2" "vgg16 16"; do
    f=gpurun_out/sanitize/${tool}_$(echo $t | tr ' ' '_')_final.log
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py $t > $f 2>&1
    echo "$tool $t rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $f | tail -1)"
  done
done | tee $E/sanitize_vgg.txt
timeout 300 python tools/profile_ops.py vgg16 256 1 > $E/ops_vgg16.txt 2>&1; head -1 $E/ops_vgg16.txt
