# ncu full capture of the FP64-pipe BConv against the IMAD.WIDE BConv (same bench workload)
mkdir -p gpurun_out
timeout 600 env CK32_BCONV_FP64=${MODE:-1} ncu --set full --import-source on --clock-control none -k regex:"k_bconv" -s 3 -c 1 -f -o gpurun_out/df python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-sweep --no-small > gpurun_out/ncu_df.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_bconv" -s 3 -c 1 -f -o gpurun_out/imad python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-sweep --no-small > gpurun_out/ncu_imad.log 2>&1
tail -2 gpurun_out/ncu_df.log gpurun_out/ncu_imad.log
