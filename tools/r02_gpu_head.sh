cd $GRAFT_REPO_ROOT
O=gpurun_out/head; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/gpu.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "rc=$?" >> $O/bench_default.err
for c in ncf lstm bert; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/bench_$c.json 2>> $O/bench_cfg.err
done
timeout 300 python bench.py --config bert --density 0.1 --no-cpu-baseline --no-e2e > $O/bench_bert10.json 2>> $O/bench_cfg.err
LHC_LIB=scratch/liblhc_ptime.so timeout 300 python tools/peel_rounds.py vgg ncf > $O/rounds.txt 2>&1
