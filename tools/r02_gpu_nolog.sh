cd $GRAFT_REPO_ROOT
O=gpurun_out/nolog; mkdir -p $O
LHC_LIB=scratch/liblhc_ptime.so timeout 300 python tools/peel_rounds.py vgg > $O/rounds.txt 2>&1
LHC_LIB=scratch/liblhc_nolog.so timeout 300 python tools/peel_rounds.py vgg >> $O/rounds.txt 2>&1
