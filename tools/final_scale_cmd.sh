set -x
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/gpu_multi.txt 2>&1; echo "rc=$?" >> gpurun_out/gpu_multi.txt
timeout 300 python bench.py > gpurun_out/fin_n1.json 2> gpurun_out/fin_n1.err
for n in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n > gpurun_out/fin_n$n.json 2> gpurun_out/fin_n$n.err
done
echo done
