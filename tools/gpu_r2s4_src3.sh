# source-level stall sampling of the plain row passes (forward, forward + combine, inverse)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name k_row -c 4 -f -o gpurun_out/src_row4 $B > gpurun_out/src_row4.log 2>&1
tail -3 gpurun_out/src_row4.log
ls -la gpurun_out | grep src_row
