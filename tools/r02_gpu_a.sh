cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_gputest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a_gputest.txt
timeout 600 python bench.py > gpurun_out/r02a_bench_vgg.json 2> gpurun_out/r02a_bench_vgg.err; echo "bench rc=$?" >> gpurun_out/r02a_bench_vgg.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02a_vgg_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02a_ncu.log 2>&1
echo done
