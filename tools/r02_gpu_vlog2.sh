cd $GRAFT_REPO_ROOT
O=gpurun_out/vlog2; mkdir -p $O
for c in vgg ncf lstm bert; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/${c}.json 2>> $O/err.txt
done
timeout 300 python bench.py --config bert --density 0.1 --no-cpu-baseline --no-e2e > $O/bert10.json 2>> $O/err.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "full_size or pipeline or cell_build or blocked or overflow or empty" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
