cd $GRAFT_REPO_ROOT
O=gpurun_out/fm; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_guards.py -q -p no:cacheprovider > $O/guards.txt 2>&1; echo "rc=$?" >> $O/guards.txt
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > $O/gpu_tests_multi.txt 2>&1; echo "rc=$?" >> $O/gpu_tests_multi.txt
run() {  # name N args...
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29610 bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err
  echo "rc=$?" >> $O/$name.err
}
run n2_default 2
run n4_default 4
run n4_replicated 4 --decode replicated --no-e2e
run n4_nccl 4 --decode replicated --comm nccl --no-e2e
