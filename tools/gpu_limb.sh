# config 4 on one GPU: unsharded, then 2/4/8 virtual shards with the gather and the peer exchange
mkdir -p gpurun_out
for ex in gather peer; do for g in 0 2 4 8; do
  python bench.py --workload limb --steps 20 --warmup 3 --exchange $ex --virtual-shards $g 2>&1 | tail -1 | tee -a gpurun_out/limb.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$ex', 'shards', d['config']['shards'], 'ms/step', d['ms_per_step'], 'exact', d['bit_exact_vs_single_device'], 'launches', d['gpu_launches'])"
done; done
