set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "row8 or ntt or intt" 2>&1 | tail -3
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k={x['kernel']:(x['GBps'],x['share']) for x in d['kernels']}
print('$1', d['value'], d['bit_exact'], d['roofline']['frac'], {a:k[a] for a in ('ntt_fwd','ntt_inv','ntt_fwd+combine')})"; }
for rep in 1 2; do run CK32_ROW8=0; run CK32_ROW8=1; done
mkdir -p gpurun_out
CK32_ROW8=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem --clock-control none -k regex:k_row -c 40 --csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-small --no-sweep --no-extra > gpurun_out/ncu_row8.csv 2>/dev/null
tail -5 gpurun_out/ncu_row8.csv
