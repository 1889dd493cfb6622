cd $GRAFT_REPO_ROOT
O=gpurun_out/p2u; mkdir -p $O
for v in u1 u2 u3 u4; do
  for c in vgg bert; do
    LHC_LIB=scratch/liblhc_$v.so timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_$v.json 2>> $O/err.txt
  done
done
