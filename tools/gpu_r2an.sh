# k_col_tma (CK32_COL=4): parity, standalone NTT A/B, whole-step A/B
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variant_paths and COL" 2>&1 | tail -2
for v in 3 4 3 4; do echo "COL=$v"; CK32_COL=$v timeout 120 python tools/prof_ntt.py 768 20; done
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], k['ntt_fwd'], k['ntt_inv'], k['ntt_row+keymult'])"; }
for rep in 1 2; do run CK32_COL=3; run CK32_COL=4; done
