cd $GRAFT_REPO_ROOT
O=gpurun_out/i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_guards.py -q > $O/guards.txt 2>&1; echo "rc=$?" >> $O/guards.txt
timeout 2400 python tools/fig3_sweep.py --out $O/r02_fig3.json > $O/fig3.log 2>&1; echo "rc=$?" >> $O/fig3.log
