cd $GRAFT_REPO_ROOT
O=gpurun_out/cvar2; mkdir -p $O
for rep in 1 2; do
for v in base w6 w10 w12 w16; do
  for c in vgg bert lstm; do
    LHC_LIB=scratch/liblhc_$v.so timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_${v}_r$rep.json 2>> $O/err.txt
  done
done
done
