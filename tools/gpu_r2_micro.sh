# round-2 NTT design experiments (compute skeletons) + pipe-cost probes under ncu
mkdir -p gpurun_out
./tools/microbench_ntt_r2 2000 | tee gpurun_out/microbench_ntt_r2.txt
M=sm__inst_executed_pipe_fmaheavy.sum,sm__pipe_fmaheavy_cycles_active.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fmalite_cycles_active.sum,sm__inst_executed_pipe_alu.sum,sm__pipe_alu_cycles_active.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none --csv -k regex:"k_probe|k_rowskel|k_colskel" -c 16 ./tools/microbench_ntt_r2 200 > gpurun_out/microbench_ntt_r2_ncu.csv 2>&1
ncu --metrics $M --clock-control none --csv -k regex:"k_col|k_row|k_bconv|k_tensor|k_hrot_tail" -c 12 \
  python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/ncu_pipes_r2.csv 2>&1
tail -3 gpurun_out/ncu_pipes_r2.csv
