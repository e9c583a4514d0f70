# k_row_keymult_pf (CK32_KM=5) vs the round-1 default: parity, A/B bench, ncu source capture
mkdir -p gpurun_out
CK32_KM=5 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_size or mechanisms_equal or batched or oracle_sweep or default_params" 2>&1 | tail -3
for v in 0 5 0 5; do
  CK32_KM=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:x for x in d['kernels']}
print('KM=$v', d['value'], d['bit_exact'], 'row+km', k['ntt_row+keymult']['GBps'], k['ntt_row+keymult']['share'])"
done
for v in 0 5; do
CK32_KM=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_row_keymult" -s 2 -c 1 -f -o gpurun_out/km_v$v \
  python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/ncu_km_v$v.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
