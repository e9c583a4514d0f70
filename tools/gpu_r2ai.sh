# ncu --set full with source counters of the NTT passes (768 limbs, forward + inverse)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_col|k_row' -c 4 -o gpurun_out/ntt_src python tools/prof_ntt.py 768 1 > /dev/null 2>&1
ls -la gpurun_out
