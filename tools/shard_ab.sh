# C5 on one NCCL rank (tools/sharded_bench.py), with and without the forked
# slab iteration:  bash tools/shard_ab.sh
for i in 1 2; do
  for f in 0 1; do
    echo -n "BSP_DIST_FORK=$f: "
    BSP_DIST_FORK=$f timeout 300 python tools/sharded_bench.py --world 1 --rank 0 --steps 20 --warmup 10 --no-e2e 2>/dev/null | grep RESULT | cut -c8- | python -c "import json,sys; r=json.load(sys.stdin); print(r['ms_per_iter'], 'ms/iter, setup', round(r['setup_s'], 2), 's')"
  done
done
