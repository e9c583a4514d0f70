# round-2 profile set: launch lists of the default bench workload and of a B=16 one-stream step,
# ncu --set full of every hot kernel (summarised on the box; the report itself stays there)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default_r2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_b16_r2.csv python bench.py --steps 2 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -s 30 -c 30 -f -o /tmp/r2_all_full \
  python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/ncu_all_r2.log 2>&1
python tools/ncu_summary.py /tmp/r2_all_full.ncu-rep gpurun_out/ncu_all_kernels_summary_r2.csv
for k in "k_col<0, 0, 1, 5, 8, 1>" "k_row<0, 0>" "k_row<0, 3>" "k_row_keymult" "k_bconv<8>"; do
  f=$(echo "$k" | tr -c 'a-z0-9_' '_')
  ncu -i /tmp/r2_all_full.ncu-rep --page source --csv --print-source sass -k regex:"$(echo "$k" | sed 's/[<>, ]/./g')" -c 1 2>/dev/null | head -c 3000000 > gpurun_out/src_$f.csv
done
ls -la gpurun_out/
