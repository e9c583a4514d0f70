# config 4 (limb-sharded N=2^17) bench lines on one GPU: 1 shard and virtual shards
set -x
for v in 0 2 4 8; do
  python bench.py --workload limb --steps 10 --warmup 3 --virtual-shards $v 2>&1 | tail -1
done
