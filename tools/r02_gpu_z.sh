cd $GRAFT_REPO_ROOT
O=gpurun_out/z; mkdir -p $O
for v in base bmb3 bmb4; do
  if [ $v = base ]; then L=paper_2402_07529_b200/liblhc.so; else L=scratch/liblhc_$v.so; fi
  for c in vgg lstm bert; do
    LHC_LIB=$L timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_$v.json 2>> $O/err.txt
  done
done
LHC_LIB=paper_2402_07529_b200/liblhc.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_pair|k_build" -c 10 --csv --log-file $O/build_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
LHC_LIB=scratch/liblhc_bmb3.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_pair|k_build" -c 10 --csv --log-file $O/build_launches_bmb3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
