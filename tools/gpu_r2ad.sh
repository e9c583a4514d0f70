# whole-step A/B of the opt-in BConv / fused variants on the current default
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], d['roofline']['frac'], k)"; }
for rep in 1 2; do
  run X=0; run CK32_TC=1; run CK32_FUSED=1; run CK32_BCONV_FP64=4; run CK32_BCONV_FP64=6
done
