cd $GRAFT_REPO_ROOT
O=gpurun_out/ncusplit; mkdir -p $O
LHC_LIB=scratch/liblhc_ptime.so timeout 300 python tools/peel_rounds.py vgg > $O/rounds.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_peel|k_build_cells" -c 2 -o $O/vgg_peel python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $O/ncu_full.log 2>&1
