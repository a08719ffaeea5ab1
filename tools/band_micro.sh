cd $GRAFT_REPO_ROOT
export B2_DEV=1   # developer knobs (B2_*) honoured
for bd in 0 1; do
  export B2_BAND=$bd
  timeout 60 python tools/conv_micro.py 256 56 56 64 64 3 1
  timeout 60 python tools/conv_micro.py 256 28 28 128 128 3 1
  timeout 60 python tools/conv_micro.py 256 14 14 256 256 3 1
  timeout 60 python tools/conv_micro.py 256 7 7 512 512 3 1
  timeout 60 python tools/conv_micro.py 256 224 224 3 64 7 2
  timeout 60 python tools/conv_micro.py 16 224 224 64 64 3 1
done
