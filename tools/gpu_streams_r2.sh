run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['bit_exact'])"; }
for rep in 1 2; do run "--streams 2"; run "--streams 3 --batch 48"; run "--streams 3 --batch 33"; run "--streams 4 --batch 32"; run "--streams 4 --batch 64"; run "--streams 2 --batch 48"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k fused_hrot_tail 2>&1 | tail -2
