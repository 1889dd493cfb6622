# 4 B200: the driver's launch of bench.py at N = 2 and 4 (defaults: VGG19, sharded decode,
# e2e, cpu baseline off at N > 1), the NCCL baseline line, and the reference arm.
cd $GRAFT_REPO_ROOT
O=gpurun_out/m2; mkdir -p $O
run() {  # name N args...
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29610 bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err
  echo "rc=$?" >> $O/$name.err
}
run n2_default 2
run n4_default 4
run n2_nccl 2 --comm nccl --no-e2e
run n4_replicated 4 --decode replicated --no-e2e
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > $O/ref_n2.json 2> $O/ref_n2.err; echo "rc=$?" >> $O/ref_n2.err
echo done
