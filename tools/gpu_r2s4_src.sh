# source-level (per SASS instruction) stall sampling of the fused row pass + KeyMult and the forward column pass
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:k_row_keymult8 -c 1 -f -o gpurun_out/src_km8 $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:'k_col' -c 1 -f -o gpurun_out/src_col $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:'k_row<' -c 2 -f -o gpurun_out/src_row $B > /dev/null 2>&1
ls -la gpurun_out
