cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/v_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/v_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/v_smoke.txt
