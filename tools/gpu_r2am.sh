# subtractive Montgomery in every mont_mul / mont_reduce64: full GPU suite + bench
timeout 2400 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], d['roofline']['frac'], k)"; }
for rep in 1 2 3; do run X=0; done
