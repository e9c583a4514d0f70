# k_row with grouped multiplies: NTT parity, standalone NTT, whole step
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ntt or intt or hmult or hrot" 2>&1 | tail -2
for v in 1 2; do timeout 120 python tools/prof_ntt.py 768 20; done
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], k)"; }
for rep in 1 2; do run X=0; done
