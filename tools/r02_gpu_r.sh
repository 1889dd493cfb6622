cd $GRAFT_REPO_ROOT
O=gpurun_out/r; mkdir -p $O
for k in 1 2 4 8; do
  timeout 600 python bench.py --decode sharded --shards $k --steps 10 --no-cpu-baseline > $O/vgg_sh$k.json 2>> $O/err.txt
done
for k in 1 2 4; do
  timeout 600 python bench.py --config ncf --decode sharded --shards $k --steps 10 --no-cpu-baseline --no-e2e > $O/ncf_sh$k.json 2>> $O/err.txt
done
for k in 4 8; do
  timeout 600 python bench.py --config lstm --decode sharded --shards $k --steps 10 --no-cpu-baseline --no-e2e > $O/lstm_sh$k.json 2>> $O/err.txt
  timeout 600 python bench.py --config bert --decode sharded --shards $k --steps 10 --no-cpu-baseline --no-e2e > $O/bert_sh$k.json 2>> $O/err.txt
  timeout 600 python bench.py --config bert --density 0.1 --decode sharded --shards $((k*4)) --steps 10 --no-cpu-baseline --no-e2e > $O/bert10_sh$((k*4)).json 2>> $O/err.txt
done
