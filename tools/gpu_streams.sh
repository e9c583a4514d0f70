timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for sn in 1 2 4; do python bench.py --steps 5 --warmup 3 --batch 32 --streams $sn --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('streams=$sn', d['value'], d['hmult_ops_per_s'], d['hrot_ops_per_s'], d['gpu_launches'])"; done
