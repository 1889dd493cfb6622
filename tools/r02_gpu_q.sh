cd $GRAFT_REPO_ROOT
O=gpurun_out/q; mkdir -p $O
for v in new qold qmb4; do
  if [ $v = new ]; then L=paper_2402_07529_b200/liblhc.so; else L=scratch/liblhc_$v.so; fi
  for c in vgg ncf lstm bert; do
    LHC_LIB=$L timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_$v.json 2>> $O/err.txt
  done
  LHC_LIB=$L timeout 300 python bench.py --config bert --density 0.1 --steps 10 --no-cpu-baseline --no-e2e > $O/bert10_$v.json 2>> $O/err.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "query or pipeline or full_size" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
