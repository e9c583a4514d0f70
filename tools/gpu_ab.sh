# GPU parity suite, then bench A/B for env-var variants given as args (e.g. "CK32_UNFUSED=1")
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for v in "" "$@"; do env $v python bench.py --steps 5 --warmup 3 --batch ${B:-16} --no-cpu --no-e2e --no-sweep --no-small 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', 'value', d['value'], 'hmult', d['hmult_ops_per_s'], 'hrot', d['hrot_ops_per_s'], [(k['kernel'],k['share'],k['GBps']) for k in d['kernels']])"; done
