cd $GRAFT_REPO_ROOT
O=gpurun_out/split2; mkdir -p $O
for sp in 0 1; do
  for dn in 0.02 0.05; do
    LHC_PEEL_SPLIT=$sp timeout 300 python bench.py --config bert --density $dn --steps 10 --no-cpu-baseline --no-e2e > $O/bert${dn}_s$sp.json 2>> $O/err.txt
  done
  LHC_PEEL_SPLIT=$sp timeout 300 python bench.py --config vgg --index bitmap --steps 10 --no-cpu-baseline --no-e2e > $O/vggbm_s$sp.json 2>> $O/err.txt
done
python -c "import paper_2402_07529_b200 as l, ctypes; print(l.lib())" >> $O/err.txt 2>&1
