# k_row_keymult8 (CK32_KM=12): parity (variants + batched), whole-step A/B
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "(batched_keymult or variant_paths) and 13" 2>&1 | tail -2
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], d['roofline']['frac'], k['ntt_row+keymult'])"; }
for rep in 1 2; do run CK32_KM=8; run CK32_KM=13; done
B="python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra"
CK32_KM=13 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_row_keymult8' -s 2 -c 2 -o gpurun_out/km13 $B > /dev/null 2>&1
ls gpurun_out
