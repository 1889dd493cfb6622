cd $GRAFT_REPO_ROOT
O=gpurun_out/wq2; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -x -p no:cacheprovider > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for c in vgg ncf lstm bert; do
  timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/${c}.json 2>> $O/err.txt
done
for dd in 0.05 0.10; do
timeout 300 python bench.py --config bert --density $dd --steps 10 --no-cpu-baseline --no-e2e > $O/bert$dd.json 2>> $O/err.txt
done
