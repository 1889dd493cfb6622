cd $GRAFT_REPO_ROOT
O=gpurun_out/vlog; mkdir -p $O
for c in vgg ncf lstm bert; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/${c}.json 2>> $O/err.txt
done
timeout 300 python bench.py --config bert --density 0.1 --no-cpu-baseline --no-e2e > $O/bert10.json 2>> $O/err.txt
timeout 300 python bench.py --config vgg --index bitmap --no-cpu-baseline --no-e2e > $O/vgg_bitmap.json 2>> $O/err.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -x -p no:cacheprovider > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
