cd $GRAFT_REPO_ROOT
O=gpurun_out/u; mkdir -p $O
for c in vgg ncf lstm bert; do
  timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/$c.json 2>> $O/err.txt
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
