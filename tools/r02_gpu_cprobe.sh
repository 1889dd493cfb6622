cd $GRAFT_REPO_ROOT
O=gpurun_out/cprobe; mkdir -p $O
for v in base pol1 pol2 pol3 st3 st4; do
  echo "== $v" >> $O/probe.txt
  LHC_LIB=scratch/liblhc_$v.so timeout 300 python tools/compress_probe.py vgg >> $O/probe.txt 2>&1
done
LHC_LIB=scratch/liblhc_base.so timeout 300 python tools/compress_probe.py bert >> $O/probe.txt 2>&1
