cd $GRAFT_REPO_ROOT
O=gpurun_out/split; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cell_build_paths or threshold_sweep or full_size_configs or gamma_sweep" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for sp in 0 1; do
  for c in vgg lstm bert; do
    LHC_PEEL_SPLIT=$sp timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_s$sp.json 2>> $O/err.txt
  done
  LHC_PEEL_SPLIT=$sp timeout 300 python bench.py --config bert --density 0.1 --steps 10 --no-cpu-baseline --no-e2e > $O/bert10_s$sp.json 2>> $O/err.txt
done
LHC_PEEL_SPLIT=1 LHC_LIB=scratch/liblhc_ptime.so timeout 300 python tools/peel_rounds.py vgg > $O/rounds.txt 2>&1
