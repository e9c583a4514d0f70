# k_hrot_tail4 (scatter, 4 coefficients per thread): parity + A/B vs the gather tail
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hrot or GATHER or batched" 2>&1 | tail -2
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], k['hrot_tail'])"; }
for rep in 1 2; do run X=0; run CK32_TAIL_GATHER=1; done
