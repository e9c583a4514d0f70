timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keys.py tests/test_gpu_helr.py tests/test_bench_contract.py -q -m gpu -x 2>&1 | tail -3
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], k)"; }
for rep in 1 2; do run CK32_NO_KM_INTT=1; run X=1; done
