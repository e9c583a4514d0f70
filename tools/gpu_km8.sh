mkdir -p gpurun_out
CK32_KM=7 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py -q -m gpu -k "full_size or mechanisms_equal or batched or oracle_sweep or default_params or profile_bytes" 2>&1 | tail -3
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:x for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], {n: k[n]['GBps'] for n in ('ntt_row+keymult','ntt_fwd','bconv')})"; }
for rep in 1 2; do run CK32_KM=7; run CK32_KM=8; done
M=gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem
for v in 7 8; do CK32_KM=$v ncu --metrics $M --clock-control none --csv -k regex:"k_row_keymult" -c 2 python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/ncu_km8_v$v.csv 2>&1; done
