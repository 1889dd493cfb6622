cd $GRAFT_REPO_ROOT
O=gpurun_out/stream; mkdir -p $O
for v in stream nostream; do
  for c in vgg ncf lstm bert; do
    LHC_LIB=scratch/liblhc_$v.so timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_$v.json 2>> $O/err.txt
  done
done
LHC_LIB=scratch/liblhc_ptime.so timeout 300 python tools/peel_rounds.py vgg > $O/rounds.txt 2>&1
LHC_LIB=scratch/liblhc_ptime_nostream.so timeout 300 python tools/peel_rounds.py vgg >> $O/rounds.txt 2>&1
