# headline schedule A/B: B = 32 x 2 streams (default) vs B = 48 x 3 streams and 64 x 4, alternating
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['bit_exact'])"; }
for rep in 1 2 3; do run "--batch 32 --streams 2"; run "--batch 48 --streams 3"; run "--batch 64 --streams 4"; done
