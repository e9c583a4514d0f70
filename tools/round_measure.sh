# batch sweep, full bench line, launch list and one full ncu capture of the dominant kernels
mkdir -p gpurun_out
for b in 8 32 64; do B=$b python bench.py --steps 5 --warmup 3 --batch $b --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=$b', d['value'], d['hmult_ops_per_s'], d['hrot_ops_per_s'])"; done
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 3000 gpurun_out/bench_full.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --batch 16 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --import-source on -k regex:"k_(col|row|bconv|key_mult)" -s 12 -c 5 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 1 --batch 16 --no-cpu --no-e2e > /dev/null 2>&1
ls -la gpurun_out
