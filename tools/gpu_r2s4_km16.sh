# k_row_keymult8 KPF 7 (CK32_KM=16: the key MACs after all digits' row passes, summed per output in one
# expression): parity + A/B vs the default (KM=8) + ncu of the keymult launches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "(variant_paths and 16) or (batched_keymult and 16)" 2>&1 | tail -2 | tee gpurun_out/km16_pytest.txt
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], k['ntt_row+keymult'])"; }
for rep in 1 2; do run CK32_KM=8; run CK32_KM=16; done
for km in 8 16; do
CK32_KM=$km timeout 600 ncu --kernel-name regex:k_row_keymult8 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none --csv \
  python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/ncu_km$km.csv 2>/dev/null
done
python tools/ncu_km_table.py 8 16
CK32_KM=16 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:k_row_keymult8 -c 1 -f -o gpurun_out/src_km16 python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > /dev/null 2>&1
