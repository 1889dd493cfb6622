cd $GRAFT_REPO_ROOT
O=gpurun_out/k; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for c in vgg ncf lstm bert; do
  timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/$c.json 2>> $O/err.txt
done
timeout 300 python bench.py --config bert --density 0.1 --steps 10 --no-cpu-baseline --no-e2e > $O/bert10.json 2>> $O/err.txt
