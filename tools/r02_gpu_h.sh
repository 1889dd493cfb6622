cd $GRAFT_REPO_ROOT
O=gpurun_out/h; mkdir -p $O
for c in vgg bert lstm ncf; do
  for l2 in 1 0; do
    LHC_L2_PERSIST=$l2 timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_l2_$l2.json 2>> $O/err.txt
  done
  for v in ilp1 ilp4; do
    LHC_LIB=scratch/liblhc_$v.so timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_$v.json 2>> $O/err.txt
  done
done
timeout 300 python bench.py --config bert --density 0.1 --steps 10 --no-cpu-baseline --no-e2e > $O/bert10_l2_1.json 2>> $O/err.txt
LHC_L2_PERSIST=0 timeout 300 python bench.py --config bert --density 0.1 --steps 10 --no-cpu-baseline --no-e2e > $O/bert10_l2_0.json 2>> $O/err.txt
