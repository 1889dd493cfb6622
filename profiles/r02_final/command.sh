cd $GRAFT_REPO_ROOT
O=gpurun_out/final4; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/gpu.txt
lscpu > $O/lscpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/tests_gpu.txt 2>&1; echo "rc=$?" >> $O/tests_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "rc=$?" >> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for c in ncf lstm bert; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/bench_$c.json 2>> $O/bench_cfg.err
done
for dd in 0.02 0.05 0.10; do
  timeout 300 python bench.py --config bert --density $dd --no-cpu-baseline --no-e2e > $O/bench_bert_$dd.json 2>> $O/bench_cfg.err
done
for w in 2 4; do
  timeout 300 python bench.py --config bert --workers $w --no-cpu-baseline --no-e2e > $O/bench_bert_w$w.json 2>> $O/bench_cfg.err
done
timeout 300 python bench.py --deterministic --no-cpu-baseline --no-e2e > $O/bench_vgg_det.json 2>> $O/bench_cfg.err
timeout 300 python bench.py --per-worker --no-cpu-baseline --no-e2e > $O/bench_vgg_perworker.json 2>> $O/bench_cfg.err
LHC_LIB=scratch/liblhc_ptime.so timeout 300 python tools/peel_rounds.py vgg ncf lstm > $O/rounds.txt 2>&1
timeout 300 python bench.py --index bitmap --no-cpu-baseline --no-e2e > $O/bench_vgg_bitmap.json 2>> $O/bench_cfg.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/vgg_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_clear|k_compress_rows|k_query|k_pair|k_build_cells|k_peel" -c 8 -o $O/vgg_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $O/ncu_full.log 2>&1
echo done
