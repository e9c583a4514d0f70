# round-2 re-entry check: full GPU suite on HEAD (BConv on tcgen05 by default), default bench line, KeyMult variant A/B
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -6
timeout 600 python bench.py > gpurun_out/bench_default_r2ag.json 2> gpurun_out/bench_default_r2ag.err; tail -c 600 gpurun_out/bench_default_r2ag.json
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], d['roofline']['frac'], k['ntt_row+keymult'], k['bconv'])"; }
for rep in 1 2; do run X=0; run CK32_KM=9; run CK32_KM=10; run CK32_KM=11; done
