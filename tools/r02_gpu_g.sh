# Round-2 measurement batch on one B200 (tests, bench lines, ncu, sanitizers).
cd $GRAFT_REPO_ROOT
O=gpurun_out/g
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.txt
timeout 900 python bench.py > $O/bench_vgg.json 2> $O/bench_vgg.err; echo "rc=$?" >> $O/bench_vgg.err
for c in ncf lstm bert; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/bench_$c.json 2>> $O/bench_cfg.err
done
for dd in 0.02 0.05 0.10; do
  timeout 600 python bench.py --config bert --density $dd --no-cpu-baseline --no-e2e > $O/bench_bert_$dd.json 2>> $O/bench_cfg.err
done
for w in 2 4; do
  timeout 600 python bench.py --config bert --workers $w --no-cpu-baseline --no-e2e > $O/bench_bert_w$w.json 2>> $O/bench_cfg.err
done
timeout 600 python bench.py --deterministic --no-cpu-baseline --no-e2e > $O/bench_vgg_det.json 2>> $O/bench_cfg.err
timeout 600 python bench.py --per-worker --no-cpu-baseline --no-e2e > $O/bench_vgg_perworker.json 2>> $O/bench_cfg.err
timeout 600 python bench.py --index bitmap --no-cpu-baseline --no-e2e > $O/bench_vgg_bitmap.json 2>> $O/bench_cfg.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/vgg_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_clear|k_compress_dense|k_query|k_pair|k_build_cells|k_peel" -c 8 -o $O/vgg_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $O/ncu_full.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py tiny > $O/sanitize_${t}_tiny.txt 2>&1; echo "rc=$?" >> $O/sanitize_${t}_tiny.txt
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py 1m > $O/sanitize_memcheck_1m.txt 2>&1; echo "rc=$?" >> $O/sanitize_memcheck_1m.txt
timeout 1200 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py 1m > $O/sanitize_racecheck_1m.txt 2>&1; echo "rc=$?" >> $O/sanitize_racecheck_1m.txt
echo done
