mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_limb.py -q -m gpu 2>&1 | tail -3
CK32_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --workload limb --gpus 2 --steps 5 --warmup 3 2>&1 | grep -E "^\{|\[bench\]|Error|error" | cut -c1-900
CK32_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-sweep --no-small --no-extra 2>&1 | grep -E "^\{|\[bench\]|Error|error" | cut -c1-600
timeout 300 python bench.py --workload limb --virtual-shards 8 --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-900
