cd $GRAFT_REPO_ROOT
O=gpurun_out/crows; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "compress or pipeline or generic_k or full_size_configs or negative_zero" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 300 python tools/compress_probe.py vgg > $O/probe.txt 2>&1
LHC_COMPRESS_IMPL=chunks timeout 300 python tools/compress_probe.py vgg >> $O/probe.txt 2>&1
for c in vgg ncf lstm bert; do
  timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}.json 2>> $O/err.txt
done
timeout 300 python bench.py --config bert --density 0.1 --steps 10 --no-cpu-baseline --no-e2e > $O/bert10.json 2>> $O/err.txt
