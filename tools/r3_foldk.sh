# residual fold threshold on BERT (O-projection K = 768: folded by default)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  AB_LABEL=default timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab_fk.txt 2>&1
  B2_DEV=1 B2_FOLD_MAX_K=512 AB_LABEL=fold512 timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab_fk.txt 2>&1
  B2_DEV=1 B2_FOLD_MAX_K=0 AB_LABEL=fold0 timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab_fk.txt 2>&1
done
sort -k1,1 -s gpurun_out/ab_fk.txt | grep -v "^ \|Trace\|File"
B2_DEV=1 B2_FOLD_MAX_K=512 timeout 300 python tools/profile_ops.py bert 128 2>&1 | sed -n 2,9p
