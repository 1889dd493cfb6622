cd $GRAFT_REPO_ROOT
O=gpurun_out/persist2; mkdir -p $O
for v in base nohint; do
  for pf in 1.0 0; do
    if [ $v = nohint ] && [ $pf = 0 ]; then continue; fi
    if [ $v = base ]; then L=paper_2402_07529_b200/liblhc.so; else L=scratch/liblhc_$v.so; fi
    for c in vgg ncf lstm bert; do
      LHC_LIB=$L LHC_L2_PERSIST=$pf timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_${v}_p$pf.json 2>> $O/err.txt
    done
    LHC_LIB=$L LHC_L2_PERSIST=$pf timeout 300 python bench.py --config bert --density 0.1 --steps 10 --no-cpu-baseline --no-e2e > $O/bert10_${v}_p$pf.json 2>> $O/err.txt
  done
done
LHC_L2_PERSIST=0.5 timeout 300 python bench.py --config vgg --steps 10 --no-cpu-baseline --no-e2e > $O/vgg_base_p0.5.json 2>> $O/err.txt
