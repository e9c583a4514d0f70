# column-pass attribution: k_col_tma with global stores and/or TMA loads removed (CK32_COL_DBG; timing only)
mkdir -p gpurun_out
for d in 0 1 2 3; do
  CK32_COL=4 CK32_COL_DBG=$d timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_col_tma -c 4 --csv --log-file gpurun_out/coldbg_$d.csv python tools/prof_ntt.py 768 1 > /dev/null 2>&1
done
