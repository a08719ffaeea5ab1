cd $GRAFT_REPO_ROOT
export B2_DEV=1   # developer knobs (B2_*) honoured
for cfg in "256 56 56 128 128 3 2" "256 28 28 256 256 3 2" "256 14 14 512 512 3 2"; do
  python tools/conv_micro.py $cfg; B2_PAIR=0 python tools/conv_micro.py $cfg; B2_PAIR=0 B2_FORCE_BN=256 python tools/conv_micro.py $cfg
done
