# TMA column pass (CK32_COL=3) vs cp.async (default 2): parity, standalone NTT passes, bench
mkdir -p gpurun_out
CK32_COL=3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "ntt or full_size or mechanisms_equal or batched or oracle_sweep or intt" 2>&1 | tail -3
for v in 2 3 2 3; do echo "COL=$v"; CK32_COL=$v python tools/prof_ntt.py 768 10; done
for v in 2 3 2 3; do
  CK32_COL=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:x for x in d['kernels']}
print('COL=$v', d['value'], d['bit_exact'], {n: k[n]['GBps'] for n in ('ntt_fwd','ntt_inv','ntt_fwd+combine','ntt_row+keymult')})"
done
M=sm__inst_executed_pipe_fmaheavy.sum,sm__pipe_fmaheavy_cycles_active.sum,smsp__inst_executed.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for v in 2 3; do CK32_COL=$v ncu --metrics $M --clock-control none --csv -k regex:"k_col" -c 2 python tools/prof_ntt.py 768 1 > gpurun_out/ncu_col_v$v.csv 2>&1; done
./tools/microbench_ntt_r2 200 > /dev/null
ncu --metrics $M --clock-control none --csv -k regex:"k_probe" -c 3 ./tools/microbench_ntt_r2 200 > gpurun_out/microbench_probe_ncu.csv 2>&1
