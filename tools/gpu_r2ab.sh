timeout 1700 python -m pytest tests -q -m gpu 2>&1 | tail -3
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], d['roofline']['frac'], k['ntt_row+keymult'])"; }
for rep in 1 2; do run CK32_KM=7; run CK32_KM=8; done
