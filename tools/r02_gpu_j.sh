cd $GRAFT_REPO_ROOT
O=gpurun_out/j; mkdir -p $O
for c in vgg bert lstm ncf; do
  for il in 1 0; do
    LHC_COMPRESS_INTERLEAVE=$il timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}_il$il.json 2>> $O/err.txt
  done
done
for dd in 0.05 0.10; do
  for il in 1 0; do
    LHC_COMPRESS_INTERLEAVE=$il timeout 300 python bench.py --config bert --density $dd --steps 10 --no-cpu-baseline --no-e2e > $O/bert${dd}_il$il.json 2>> $O/err.txt
  done
done
LHC_LIB=scratch/liblhc_nodense.so timeout 300 python tools/peel_diag.py vgg ncf > $O/nodense.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "compress" > $O/tests_compress.txt 2>&1
