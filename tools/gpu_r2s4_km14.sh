# k_row_keymult8 KPF 5 (CK32_KM=14: the next item's extension rows requested into each digit buffer as soon
# as the current item frees it): parity + A/B vs the default (KM=8) + ncu of one B=16 step's keymult launches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "KM=14 or batched_keymult_variants" 2>&1 | tail -2
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], k['ntt_row+keymult'])"; }
for rep in 1 2; do run CK32_KM=8; run CK32_KM=14; done
for km in 8 14; do
CK32_KM=$km timeout 600 ncu --kernel-name regex:k_row_keymult8 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none --csv \
  python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/ncu_km$km.csv 2>/dev/null
done
python - <<'PY'
import csv,io
for km in (8,14):
    txt=open(f'gpurun_out/ncu_km{km}.csv').read(); txt=txt[txt.index('"ID"'):]
    rows=list(csv.DictReader(io.StringIO(txt)))
    by={}
    for r in rows: by.setdefault(r['ID'],{})[r['Metric Name']]=r['Metric Value']
    for i,m in list(by.items())[:4]: print(km, i, {k.split('.')[0][-28:]:v for k,v in m.items()})
PY
