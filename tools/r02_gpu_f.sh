cd $GRAFT_REPO_ROOT
python tools/peel_diag.py vgg bert lstm > gpurun_out/diag11.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cell_build or full_size" > gpurun_out/r02f_gputest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02f_gputest.txt
