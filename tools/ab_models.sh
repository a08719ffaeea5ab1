# A/B: per-op profiles of the four big models, new library vs ab/libb2_base.so (HEAD)
cd $GRAFT_REPO_ROOT
for m in "resnet50 256" "bert 128" "vgg16 256" "mobilenet_v2 256"; do
  python tools/profile_ops.py $m > gpurun_out/new_${m%% *}.log 2>&1
  B2_LIB=ab/libb2_base.so python tools/profile_ops.py $m > gpurun_out/base_${m%% *}.log 2>&1
done
