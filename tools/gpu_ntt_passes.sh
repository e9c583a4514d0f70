# per-pass NTT timing: event-timed full transforms + ncu launch list of the passes
mkdir -p gpurun_out
python tools/prof_ntt.py 768 5
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ntt_passes.csv python tools/prof_ntt.py 768 2 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/ntt_passes.csv 2>&1 | head -20
