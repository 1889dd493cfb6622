cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_peel_rows -c 1 -o gpurun_out/r02_rows_ncf python tools/peel_diag.py ncf > gpurun_out/r02_ncu_rows.log 2>&1
