cd $GRAFT_REPO_ROOT
O=gpurun_out/build; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cell_build_paths or full_size_configs or threshold_sweep or blocked" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for v in b4 b3; do
  for c in vgg lstm bert; do
    LHC_LIB=scratch/liblhc_$v.so timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_$v.json 2>> $O/err.txt
  done
  LHC_LIB=scratch/liblhc_$v.so timeout 300 python bench.py --config bert --density 0.1 --steps 10 --no-cpu-baseline --no-e2e > $O/bert10_$v.json 2>> $O/err.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_build" -c 6 --csv --log-file $O/build_b4.csv python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
LHC_LIB=scratch/liblhc_b3.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_build" -c 6 --csv --log-file $O/build_b3.csv python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
