# One round-measurement call: GPU parity suite, smoke, default bench line,
# launch list (time + DRAM bytes) of a bench step, and --set full captures of
# the NTT passes (tools/prof_ntt.py) and of the fused row+KeyMult / BConv kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
SMOKE=1 timeout 300 python __graft_entry__.py 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 600 gpurun_out/bench_default.json
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep > /dev/null 2>&1
# launch list of the default bench workload itself (B = 32, 2 streams), serialised by ncu
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_(col|row)$" -c 4 -f -o gpurun_out/ntt_full \
  python tools/prof_ntt.py 768 1 > gpurun_out/ncu_ntt.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(row_keymult|bconv)" -s 6 -c 3 -f -o gpurun_out/mech_full \
  python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep > gpurun_out/ncu_mech.log 2>&1
fi
ls -la gpurun_out
