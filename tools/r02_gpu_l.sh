cd $GRAFT_REPO_ROOT
O=gpurun_out/l; mkdir -p $O
for v in base minb3 minb4 thr256 thr1024; do
  if [ $v = base ]; then L=paper_2402_07529_b200/liblhc.so; else L=scratch/liblhc_$v.so; fi
  LHC_LIB=$L timeout 600 python tools/peel_diag.py vgg ncf lstm bert > $O/$v.txt 2>&1
done
