# session-4 measurement set (current defaults): full GPU suite, default bench line, launch lists,
# ncu --set full summary of one B=16 HMult+HRot step
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4f_gputests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4f_gputests.log
timeout 900 python bench.py > gpurun_out/s4f_bench.json 2> gpurun_out/s4f_bench.err
python -c "import json; d=json.loads(open('gpurun_out/s4f_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['bit_exact'], d['roofline']['frac'], d['roofline_ntt']['frac'], d['clocks'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4f_launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/s4f_launches_b16.csv python bench.py --steps 2 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -s 30 -c 30 -f -o /tmp/s4f_full \
  python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/s4f_ncu_all.log 2>&1
python tools/ncu_summary.py /tmp/s4f_full.ncu-rep gpurun_out/s4f_ncu_all_kernels_summary.csv
ls -la gpurun_out | tail -8
