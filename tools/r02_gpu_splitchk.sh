cd $GRAFT_REPO_ROOT
O=gpurun_out/splitchk; mkdir -p $O
for sp in 0 1; do
  LHC_PEEL_SPLIT=$sp timeout 300 python bench.py --config lstm --steps 10 --no-cpu-baseline --no-e2e > $O/lstm_s$sp.json 2>> $O/err.txt
  LHC_PEEL_SPLIT=$sp timeout 300 python bench.py --config bert --density 0.05 --steps 10 --no-cpu-baseline --no-e2e > $O/bert5_s$sp.json 2>> $O/err.txt
done
