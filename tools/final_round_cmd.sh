set -x
nvidia-smi -L
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.txt
timeout 300 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
timeout 300 python bench.py --config vgg --no-cpu-baseline > gpurun_out/bench_vgg.json 2> gpurun_out/bench_vgg.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1
echo done
