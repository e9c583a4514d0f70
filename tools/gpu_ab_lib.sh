# whole-library A/B: the working tree's _lib/libck32b200.so ("new") vs _lib_ab/base.so ("base"),
# alternating default bench runs; per-kernel ncu durations of one B=16 step for both
mkdir -p gpurun_out
L=paper_2407_13055_b200/_lib
cp $L/libck32b200.so /tmp/new.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "${PYTEST_K:-hmult or hrot or intt or batched}" 2>&1 | tail -2
run() { cp /tmp/$1.so $L/libck32b200.so; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(round(x['GBps']),round(x['share'],4)) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], k)"; }
cp paper_2407_13055_b200/_lib_ab/base.so /tmp/base.so
for rep in 1 2; do run new; run base; done
for v in new base; do
  cp /tmp/$v.so $L/libck32b200.so
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_launch_$v.csv \
    python bench.py --steps 1 --warmup 1 --batch 16 --streams 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > /dev/null 2>&1
done
cp /tmp/new.so $L/libck32b200.so
python tools/launch_table.py gpurun_out/ab_launch_new.csv 2>/dev/null | head -14
python tools/launch_table.py gpurun_out/ab_launch_base.csv 2>/dev/null | head -14
