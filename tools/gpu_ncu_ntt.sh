# full ncu capture of the four NTT pass kernels on the prof_ntt workload
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"k_(col|row)" -c 4 -o gpurun_out/ntt_full -f python tools/prof_ntt.py 768 1 > gpurun_out/ncu_ntt.log 2>&1
tail -3 gpurun_out/ncu_ntt.log
