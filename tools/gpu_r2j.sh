mkdir -p gpurun_out
timeout 1700 python -m pytest tests -q -m gpu 2>&1 | tail -4
SMOKE=1 timeout 300 python __graft_entry__.py 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -3 gpurun_out/bench_default.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
for k in ['value','bit_exact','roofline','roofline_ntt','e2e','config4_limb_n131072','config5_helr','single_ciphertext']:
    print(k, json.dumps(d.get(k))[:400])
print(json.dumps(d['kernels']))
PY
python tools/pcie_bw.py
