cd $GRAFT_REPO_ROOT
O=gpurun_out/wq; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cell_build_paths or threshold_sweep or full_size_configs or compress" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for c in vgg bert; do
  timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}.json 2>> $O/err.txt
done
timeout 300 python bench.py --config bert --density 0.02 --steps 10 --no-cpu-baseline --no-e2e > $O/bert2.json 2>> $O/err.txt
timeout 300 python bench.py --per-worker --steps 10 --no-cpu-baseline --no-e2e > $O/vgg_perworker.json 2>> $O/err.txt
LHC_LIB=scratch/liblhc_ptime.so timeout 300 python tools/peel_rounds.py vgg > $O/rounds.txt 2>&1
