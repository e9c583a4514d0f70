# tc2 issue-group cache + subtractive Montgomery in k_row_keymult8: parity + bench
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], d['roofline']['frac'], k['ntt_row+keymult'], k['bconv'])"; }
for rep in 1 2 3; do run X=0; done
