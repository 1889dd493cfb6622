cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/tests_gpu.txt 2>&1; echo "rc=$?" >> $O/tests_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "rc=$?" >> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --deterministic --no-cpu-baseline > $O/bench_det.json 2> $O/bench_det.err
for c in ncf lstm bert; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench_cfg.err
done
timeout 300 python bench.py --config bert --density 0.1 --no-cpu-baseline > $O/bench_bert10.json 2>> $O/bench_cfg.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
