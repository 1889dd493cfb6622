cd $GRAFT_REPO_ROOT
O=gpurun_out/cprobe4; mkdir -p $O
for v in w4 w12 w16; do
echo "== $v" >> $O/probe.txt
LHC_LIB=scratch/liblhc_$v.so timeout 300 python tools/compress_probe.py vgg >> $O/probe.txt 2>&1
done
LHC_LIB=scratch/liblhc_base.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_compress_dense" -c 2 -o $O/vgg_compress python tools/compress_probe.py vgg > $O/ncu.log 2>&1
