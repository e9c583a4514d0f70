# CK32_COL=5: the TMA column pass register-capped at 80 for 6 CTAs / SM, parity + A/B vs the default (3)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variant_paths and COL=5" 2>&1 | tail -2
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(round(x['GBps']),round(x['share'],4)) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], k['ntt_fwd'], k['ntt_inv'])"; }
for rep in 1 2; do run CK32_COL=3; run CK32_COL=5; done
for v in 3 5; do CK32_COL=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/col_launch_$v.csv \
    python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/col_launch_$v.csv 2>/dev/null | grep k_col; done
