# 4 B200, final round-2 state: multi-GPU parity suite, the driver's launch at N = 2 and 4
# (defaults: VGG19, sharded decode, e2e), replicated P2P / NCCL baselines, the reference arm.
cd $GRAFT_REPO_ROOT
O=gpurun_out/m3; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > $O/gpu_tests_multi.txt 2>&1; echo "rc=$?" >> $O/gpu_tests_multi.txt
run() {  # name N args...
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29610 bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err
  echo "rc=$?" >> $O/$name.err
}
run n2_default 2
run n4_default 4
run n2_replicated 2 --decode replicated --no-e2e
run n4_replicated 4 --decode replicated --no-e2e
run n2_nccl 2 --decode replicated --comm nccl --no-e2e
run n4_nccl 4 --decode replicated --comm nccl --no-e2e
run n4_sharded_nvls 4 --comm nvls --no-e2e
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > $O/ref_n2.json 2> $O/ref_n2.err; echo "rc=$?" >> $O/ref_n2.err
echo done
