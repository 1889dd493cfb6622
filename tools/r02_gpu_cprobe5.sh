cd $GRAFT_REPO_ROOT
O=gpurun_out/cprobe5; mkdir -p $O
for pf in 1.0 0.5; do
echo "== persist $pf" >> $O/probe.txt
PERSIST=$pf timeout 300 python tools/compress_probe.py vgg >> $O/probe.txt 2>&1
done
echo "== bert" >> $O/probe.txt
timeout 300 python tools/compress_probe.py bert >> $O/probe.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_compress_rows" -c 1 -o $O/vgg_compress python tools/compress_probe.py vgg > $O/ncu.log 2>&1
