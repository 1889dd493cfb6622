cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02b_gputest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_gputest.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02b_bench_vgg.json 2> gpurun_out/r02b_bench_vgg.err; echo "bench rc=$?" >> gpurun_out/r02b_bench_vgg.err
timeout 300 python bench.py --config ncf --no-cpu-baseline --no-e2e > gpurun_out/r02b_bench_ncf.json 2>> gpurun_out/r02b_bench_vgg.err
echo done
