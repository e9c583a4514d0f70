# ncu --set full + source counters of the default step's hot kernels (B = 16, one stream)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_row_keymult8|k_bconv_tc|k_hrot_tail|k_tensor' -s 12 -c 8 -o gpurun_out/step_a $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_row|k_col' -s 40 -c 14 -o gpurun_out/step_b $B > /dev/null 2>&1
ls -la gpurun_out
