cd $GRAFT_REPO_ROOT
O=gpurun_out/probe; mkdir -p $O
for c in vgg lstm bert; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/${c}_base.json 2>> $O/err.txt
  LHC_PEEL_BY_PROBE=1 timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/${c}_probe.json 2>> $O/err.txt
done
LHC_PEEL_BY_PROBE=1 timeout 300 python bench.py --config bert --density 0.1 --no-cpu-baseline --no-e2e > $O/bert10_probe.json 2>> $O/err.txt
LHC_PEEL_BY_PROBE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "full_size or pipeline or cell_build or overflow or empty" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
