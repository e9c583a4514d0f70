mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_bconv_tc" -s 3 -c 2 -f -o gpurun_out/tc python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e > gpurun_out/ncu_tc.log 2>&1
tail -3 gpurun_out/ncu_tc.log
