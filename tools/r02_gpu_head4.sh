# 4 B200 at HEAD: the whole GPU suite (single- and multi-GPU tests), smoke, and the
# driver's launches at N = 1, 2, 4.
cd $GRAFT_REPO_ROOT
O=gpurun_out/h4; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/tests_gpu.txt 2>&1; echo "rc=$?" >> $O/tests_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 600 python bench.py > $O/n1_default.json 2> $O/n1_default.err; echo "rc=$?" >> $O/n1_default.err
run() {  # name N args...
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29610 bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err
  echo "rc=$?" >> $O/$name.err
}
run n2_default 2
run n4_default 4
