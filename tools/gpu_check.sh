# quick GPU check: parity suite + one bench line summary
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --batch ${B:-16} --no-cpu --no-e2e --no-sweep --no-small 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'hmult', d['hmult_ops_per_s'], 'hrot', d['hrot_ops_per_s'], [(k['kernel'],k['share'],k['GBps']) for k in d['kernels']])"
