cd $GRAFT_REPO_ROOT
O=gpurun_out/cprobe3; mkdir -p $O
echo "== base" >> $O/probe.txt
LHC_LIB=scratch/liblhc_base.so timeout 300 python tools/compress_probe.py vgg >> $O/probe.txt 2>&1
echo "== base interleave" >> $O/probe.txt
LHC_COMPRESS_INTERLEAVE=1 LHC_LIB=scratch/liblhc_base.so timeout 300 python tools/compress_probe.py vgg >> $O/probe.txt 2>&1
