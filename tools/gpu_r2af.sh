timeout 2000 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], d['roofline']['frac'], k['ntt_row+keymult'], k['bconv'])"; }
for rep in 1 2 3; do run X=0; run CK32_TC=0; run CK32_KM=11; done
