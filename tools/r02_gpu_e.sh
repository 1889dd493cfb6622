cd $GRAFT_REPO_ROOT
python tools/peel_diag.py ncf vgg > gpurun_out/diag10.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pipeline or deterministic or full_size or threshold or table1 or gamma" > gpurun_out/r02e_gputest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02e_gputest.txt
