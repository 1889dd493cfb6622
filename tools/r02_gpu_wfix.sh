cd $GRAFT_REPO_ROOT
O=gpurun_out/wfix; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_multi.py -q -p no:cacheprovider -k "compress or guard or pipeline or sharded or multi" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 600 python bench.py > $O/n1_default.json 2> $O/n1_default.err; echo "rc=$?" >> $O/n1_default.err
run() {  # name N args...
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29610 bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err
  echo "rc=$?" >> $O/$name.err
}
run n2_default 2
run n4_default 4
