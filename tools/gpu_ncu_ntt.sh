# full ncu capture of the four NTT pass kernels on the prof_ntt workload (768 limbs)
mkdir -p gpurun_out
python tools/prof_ntt.py 768 5
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_(col|row)" -c 4 -f -o gpurun_out/ntt_full python tools/prof_ntt.py 768 1 > gpurun_out/ncu_ntt.log 2>&1
tail -2 gpurun_out/ncu_ntt.log
