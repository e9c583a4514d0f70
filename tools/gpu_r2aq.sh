# k_bconv_tc2: simpler source-tile issue, immediate-offset stores for consecutive destination rows
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bconv or mechanism or hmult or hrot or batched" 2>&1 | tail -2
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], k['bconv'])"; }
for rep in 1 2 3; do run X=0; done
B="python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_bconv_tc' -s 6 -c 4 -o gpurun_out/tc2b $B > /dev/null 2>&1
