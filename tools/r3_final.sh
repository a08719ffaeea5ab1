# final round evidence: the r3 evidence refresh, then both compute-sanitizer matrices
cd $GRAFT_REPO_ROOT
bash tools/r3_evidence.sh
bash tools/sanitize.sh > gpurun_out/ev/sanitize1.txt 2>&1
bash tools/r3_sanitize2.sh > gpurun_out/ev/sanitize2.txt 2>&1
cat gpurun_out/ev/sanitize1.txt gpurun_out/ev/sanitize2.txt
