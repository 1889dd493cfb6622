set -x
for c in ncf vgg; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_query -c 1 -f -o gpurun_out/query_$c python bench.py --config $c --no-cpu-baseline --no-e2e --no-graph --steps 2 --warmup 3 > gpurun_out/ncu_query_$c.log 2>&1
done
for c in ncf lstm bert; do
timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
timeout 300 python bench.py --config bert --density 0.1 --steps 5 --warmup 5 --no-cpu-baseline > gpurun_out/cfg_bert10.json 2> gpurun_out/cfg_bert10.err
echo done
