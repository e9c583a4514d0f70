run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], d['roofline']['frac'], k['ntt_row+keymult'], k['bconv'])"; }
for rep in 1 2 3; do
  run CK32_KM=8; run CK32_KM=9; run CK32_KM=10; run CK32_TC=1
done
for v in 8 9 10; do
CK32_KM=$v timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:k_row_keymult -c 4 --csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | grep k_row_keymult | awk -F'","' -v v=$v '{print "KM=" v, $13, $15}'
done
