cd $GRAFT_REPO_ROOT
O=gpurun_out/f0; mkdir -p $O
LHC_LIB=scratch/liblhc_ptime_f0.so timeout 600 python tools/peel_rounds.py vgg ncf lstm bert > $O/rounds.txt 2>&1
for v in base bmb2; do
  if [ $v = base ]; then L=paper_2402_07529_b200/liblhc.so; else L=scratch/liblhc_$v.so; fi
  for c in vgg ncf lstm bert; do
    LHC_LIB=$L timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/${c}_$v.json 2>> $O/err.txt
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -x -p no:cacheprovider > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
