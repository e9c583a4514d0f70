# ALU-pinned butterfly adds (new lib) vs HEAD (base), + e2e with the NUMA pinning at N=1
nvidia-smi topo -m 2>/dev/null | head -4
PYTEST_K="hmult or hrot or intt or batched or ntt" bash tools/gpu_ab_lib.sh
for rep in 1 2; do timeout 600 python bench.py --no-cpu --no-small --no-sweep --no-extra 2>gpurun_out/alu_e2e.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('e2e', d['value'], d['e2e']['value'])"; done
grep NUMA gpurun_out/alu_e2e.err
