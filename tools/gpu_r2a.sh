# round 2, first call: GPU parity suite + smoke + default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
SMOKE=1 timeout 300 python __graft_entry__.py 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 1500 gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
