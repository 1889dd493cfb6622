cd $GRAFT_REPO_ROOT
O=gpurun_out/cprobe2; mkdir -p $O
for pf in 1.0 0.75 0.5; do
  echo "== base persist $pf" >> $O/probe.txt
  PERSIST=$pf LHC_LIB=scratch/liblhc_base.so timeout 300 python tools/compress_probe.py vgg >> $O/probe.txt 2>&1
done
echo "== pol2 persist 1.0" >> $O/probe.txt
PERSIST=1.0 LHC_LIB=scratch/liblhc_pol2.so timeout 300 python tools/compress_probe.py vgg >> $O/probe.txt 2>&1
