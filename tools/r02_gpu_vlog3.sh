cd $GRAFT_REPO_ROOT
O=gpurun_out/vlog3; mkdir -p $O
LHC_LIB=scratch/liblhc_ptime_new.so timeout 600 python tools/peel_rounds.py vgg ncf lstm bert > $O/rounds_new.txt 2>&1
for c in vgg ncf lstm bert; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/${c}.json 2>> $O/err.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "full_size or pipeline or cell_build or blocked or overflow or empty or runtime or mask" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
