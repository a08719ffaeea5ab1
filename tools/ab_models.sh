# A/B: per-op profiles, new library vs ab/libb2_base.so (HEAD); models from $AB_MODELS
export B2_DEV=1   # developer knobs (B2_*) honoured
cd $GRAFT_REPO_ROOT
for m in ${AB_MODELS:-"resnet50:256" "bert:128" "vgg16:256" "mobilenet_v2:256"}; do
  n=${m%%:*}; b=${m##*:}
  python tools/profile_ops.py $n $b > gpurun_out/new_$n.log 2>&1
  B2_LIB=ab/libb2_base.so python tools/profile_ops.py $n $b > gpurun_out/base_$n.log 2>&1
done
