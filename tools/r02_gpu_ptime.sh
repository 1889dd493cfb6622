cd $GRAFT_REPO_ROOT
O=gpurun_out/ptime; mkdir -p $O
for v in old new; do
  LHC_LIB=scratch/liblhc_ptime_$v.so timeout 600 python tools/peel_rounds.py vgg ncf lstm bert > $O/rounds_$v.txt 2>&1
done
