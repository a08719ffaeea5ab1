cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { AB_LABEL="$1" env B2_DEV=1 $2 timeout 300 python tools/fwd_time.py resnet50 256 >> gpurun_out/ab5.log 2>&1; }
run default ""
run fold128 "B2_FOLD_MAX_K=128"
run fold0 "B2_FOLD_MAX_K=0"
run fold256 "B2_FOLD_MAX_K=256"
cat gpurun_out/ab5.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_gemm2_kernel -s 5 -c 3 -o gpurun_out/r2_full_l3 python tools/ncu_target.py resnet50 256 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python tools/elastic_c5.py gpurun_out/r2_c5 > gpurun_out/c5.log 2>&1
tail -5 gpurun_out/c5.log
