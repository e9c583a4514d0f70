# source-level stall sampling: forward + inverse column pass, row passes (one B=16 step)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:'k_col' -c 3 -f -o gpurun_out/src_col3 $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:'k_row<' -c 3 -f -o gpurun_out/src_row3 $B > /dev/null 2>&1
ls -la gpurun_out
