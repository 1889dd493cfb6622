cd $GRAFT_REPO_ROOT
O=gpurun_out/ncuf; mkdir -p $O
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain.json 2> $O/plain.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/vgg_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_compress_rows|k_peel" -c 2 -o $O/vgg_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $O/ncu_full.log 2>&1
