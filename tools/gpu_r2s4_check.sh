# session-4 re-entry check: full GPU suite + default bench line on the rebuilt library
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4_gputests.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/s4_gputests.log
timeout 900 python bench.py > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err
tail -c 600 gpurun_out/s4_bench.json
