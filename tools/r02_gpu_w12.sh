cd $GRAFT_REPO_ROOT
O=gpurun_out/w12; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -x -p no:cacheprovider -k "compress or guard or pipeline or full_size" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "rc=$?" >> $O/bench_default.err
timeout 300 python bench.py --per-worker --no-cpu-baseline --no-e2e > $O/vgg_perworker.json 2>> $O/err.txt
timeout 300 python bench.py --config ncf --no-cpu-baseline --no-e2e > $O/ncf.json 2>> $O/err.txt
timeout 300 python bench.py --config bert --density 0.1 --no-cpu-baseline --no-e2e > $O/bert10.json 2>> $O/err.txt
