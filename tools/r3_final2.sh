# after the attention softmax change: full GPU suite, BERT sanitizer runs, BERT profiles
cd $GRAFT_REPO_ROOT
E=gpurun_out/ev2; mkdir -p $E gpurun_out/sanitize
timeout 2400 python -m pytest tests -m gpu -q -rf > $E/gputests.log 2>&1; tail -2 $E/gputests.log
for tool in memcheck racecheck synccheck; do
  for t in "bert 2" "bert 32"; do
    f=gpurun_out/sanitize/${tool}_$(echo $t | tr ' ' '_')_final.log
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py $t > $f 2>&1
    echo "$tool $t rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $f | tail -1)"
  done
done | tee $E/sanitize_bert.txt
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $E/lm_bert.csv python tools/ncu_target.py bert 128 > /dev/null 2>&1
python tools/ncu_launch_table.py $E/lm_bert.csv $E/launch_table_bert.txt embed_ln > /dev/null 2>&1
timeout 300 python tools/profile_ops.py bert 128 1 > $E/ops_bert.txt 2>&1
head -1 $E/ops_bert.txt
