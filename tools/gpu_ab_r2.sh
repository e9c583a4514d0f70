# A/B of the round-2 latency variants: k_row_keymult L2 prefetch (CK32_KM=6), combine row pass early/L2 (CK32_COMB_EARLY=1/2)
mkdir -p gpurun_out
CK32_KM=6 CK32_COMB_EARLY=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_size or mechanisms_equal or batched or oracle_sweep" 2>&1 | tail -2
CK32_COMB_EARLY=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_size or mechanisms_equal or oracle_sweep" 2>&1 | tail -2
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:x for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], {n: k[n]['GBps'] for n in ('ntt_fwd','ntt_inv','ntt_fwd+combine','ntt_row+keymult','bconv')})"; }
for rep in 1 2; do
run CK32_KM=0; run CK32_KM=6; run CK32_COMB_EARLY=1; run CK32_COMB_EARLY=2
done
