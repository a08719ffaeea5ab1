# Round evidence refresh: ncu launch list -> profiles/ncu_traffic.json inputs, per-launch tables
# (ResNet-50 b=256, BERT b=128), per-model op profiles, the full GPU suite, bench line, C4 sweep.
cd $GRAFT_REPO_ROOT
E=gpurun_out/ev; mkdir -p $E
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $E/lm_r50.csv python tools/ncu_target.py resnet50 256 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $E/lm_bert.csv python tools/ncu_target.py bert 128 > /dev/null 2>&1
python tools/ncu_launch_table.py $E/lm_r50.csv $E/launch_table_resnet50.txt > /dev/null 2>&1
python tools/ncu_traffic_json.py $E/lm_r50.csv $E/ncu_traffic.json > /dev/null 2>&1
cp $E/ncu_traffic.json profiles/ncu_traffic.json   # bench.py below reads it
python tools/ncu_launch_table.py $E/lm_bert.csv $E/launch_table_bert.txt embed_ln > /dev/null 2>&1
for m in "resnet50 256" "bert 128" "vgg16 256" "mobilenet_v2 256"; do
  set -- $m; timeout 300 python tools/profile_ops.py $1 $2 1 > $E/ops_$1.txt 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q -rf > $E/gputests.log 2>&1
tail -3 $E/gputests.log
timeout 900 python bench.py > $E/bench.json 2> $E/bench.err
python -c "import json;d=json.loads(open('$E/bench.json').read());print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d.get('sweep_c4',{}).get('wall_s'))"
timeout 900 python tools/sweep_bench.py $E/sweep_c4 > $E/sweep.log 2>&1; tail -2 $E/sweep.log
# one --set full capture each of the dominant kernels (CTA-pair GEMM, chain) at the bench config
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_gemm2 -s 12 -c 1 -o $E/gemm2_full python tools/ncu_target.py resnet50 256 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:chain_gemm -s 1 -c 1 -o $E/chain_full python tools/ncu_target.py resnet50 256 > /dev/null 2>&1
ls -la $E/*.ncu-rep
