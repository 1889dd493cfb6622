cd $GRAFT_REPO_ROOT
O=gpurun_out/thr; mkdir -p $O
for v in t512 t256 t1024; do
  for c in vgg ncf lstm bert; do
    LHC_LIB=scratch/liblhc_$v.so timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_$v.json 2>> $O/err.txt
  done
done
