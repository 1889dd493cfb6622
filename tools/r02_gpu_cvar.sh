cd $GRAFT_REPO_ROOT
O=gpurun_out/cvar; mkdir -p $O
for v in base st3 w12 w4; do
  echo "== $v" >> $O/probe.txt
  LHC_LIB=scratch/liblhc_$v.so timeout 300 python tools/compress_probe.py vgg >> $O/probe.txt 2>&1
  LHC_LIB=scratch/liblhc_$v.so timeout 300 python tools/compress_probe.py bert >> $O/probe.txt 2>&1
done
