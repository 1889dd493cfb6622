cd $GRAFT_REPO_ROOT
O=gpurun_out/persist; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cell_build_paths or threshold_sweep or full_size_configs or generic_k" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for v in base nohint; do
  for pf in 1.0 0; do
    if [ $v = base ]; then L=paper_2402_07529_b200/liblhc.so; else L=scratch/liblhc_$v.so; fi
    for c in vgg ncf lstm bert; do
      LHC_LIB=$L LHC_L2_PERSIST=$pf timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_${v}_p$pf.json 2>> $O/err.txt
    done
    LHC_LIB=$L LHC_L2_PERSIST=$pf timeout 300 python bench.py --config bert --density 0.1 --steps 10 --no-cpu-baseline --no-e2e > $O/bert10_${v}_p$pf.json 2>> $O/err.txt
  done
done
LHC_L2_PERSIST=0 LHC_LIB=scratch/liblhc_ptime.so timeout 300 python tools/peel_rounds.py vgg >> $O/rounds.txt 2>&1
