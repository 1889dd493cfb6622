cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_blocked" > gpurun_out/cl_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/cl_tests.txt
timeout 600 python tools/blk_seeds.py vgg 5 1.30 1024 196608 > gpurun_out/cl_seeds_vgg.txt 2>&1
timeout 600 python bench.py --blocks auto --block-cells 196608 --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/cl_bench_vgg.json 2> gpurun_out/cl_bench_vgg.err
