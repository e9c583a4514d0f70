mkdir -p gpurun_out
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['e2e']['value'])"; }
for rep in 1 2; do run CK32_COL=3; run CK32_COL=2; run CK32_COMB_EARLY=0; done
numactl -H 2>/dev/null | head -5; nvidia-smi topo -m 2>/dev/null | head -5
CUDA_LAUNCH_BLOCKING=0 python tools/pcie_bw.py
