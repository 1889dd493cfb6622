cd $GRAFT_REPO_ROOT
python tools/peel_diag.py ncf vgg > gpurun_out/diag5.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02d_gputest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02d_gputest.txt
