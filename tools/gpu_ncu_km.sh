mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_row_keymult" -s 2 -c 1 -f -o gpurun_out/km2 python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e > /dev/null 2>&1
ls gpurun_out
