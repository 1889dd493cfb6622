# Multi-GPU batch (4 B200): parity tests at world 2/4, bench lines N = 2/4 on VGG19.
cd $GRAFT_REPO_ROOT
O=gpurun_out/m; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_multi.py -q > $O/gpu_tests_multi.txt 2>&1; echo "rc=$?" >> $O/gpu_tests_multi.txt
run() {  # name N args...
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err
  echo "rc=$?" >> $O/$name.err
}
for n in 2 4; do
  run vgg_n${n}_p2p $n
  run vgg_n${n}_nvls $n --comm nvls --no-e2e
  run vgg_n${n}_nccl $n --comm nccl --no-e2e
  run vgg_n${n}_sharded $n --decode sharded --no-e2e
  run vgg_n${n}_sharded_nvls $n --decode sharded --comm nvls --no-e2e
  run ncf_n${n}_p2p $n --config ncf --no-e2e
done
echo done
