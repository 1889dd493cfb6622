cd $GRAFT_REPO_ROOT
O=gpurun_out/n; mkdir -p $O
for c in vgg lstm bert; do
  for z in 1 0; do
    LHC_ZERO_FIRST=$z timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_z$z.json 2>> $O/err.txt
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or cell_build or pipeline" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
