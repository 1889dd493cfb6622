cd $GRAFT_REPO_ROOT
O=gpurun_out/y; mkdir -p $O
for v in base norehash; do
  if [ $v = base ]; then L=paper_2402_07529_b200/liblhc.so; else L=scratch/liblhc_$v.so; fi
  for c in vgg ncf lstm bert; do
    LHC_LIB=$L timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_$v.json 2>> $O/err.txt
  done
done
