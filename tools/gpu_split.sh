run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['bit_exact'], d['ms_per_step'])"; }
for rep in 1 2; do run "--split batch"; run "--split ops"; run "--split ops --batch 16"; run "--split batch --batch 64"; run "--split ops --batch 64"; done
