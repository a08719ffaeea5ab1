cd $GRAFT_REPO_ROOT
cat > /tmp/t.py <<'PY'
import sys
sys.path.insert(0, ".")
from paper_2006_05096_b200 import plan as P, runtime as R, zoo
plan = R.Plan(zoo.build_plan("mlp", P.DT_BF16), P.DT_BF16)
plan.bench(4, n=3, warmup=1)
plan.profile_ops(4, iters=1)
plan.close()
print("nvtx-target ok")
PY
for inc in "b2.bench*/" "regex:b2.bench.*/" "b2.bench b=4 warmup=1 n=3/" "op 1 kind*/" "no-such*/"; do
  n=$(timeout 300 ncu --nvtx --nvtx-include "$inc" --metrics gpu__time_duration.sum --csv python /tmp/t.py 2>&1 | grep -c gpu__time_duration)
  echo "[$inc] -> $n"
done
