cd $GRAFT_REPO_ROOT
for m in 0 1 2 4 7; do echo "== LHC_ROWS_DBG=$m"; LHC_ROWS_DBG=$m python tools/peel_diag.py ncf 2>&1 | grep -E "peel \(all|round (2|10):"; done > gpurun_out/diag8.txt
