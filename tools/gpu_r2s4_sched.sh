# whole-step schedule sweep: batch per step x streams (default kernels)
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['ms_per_step'], d['bit_exact'])"; }
for a in "--batch 32 --streams 2" "--batch 32 --streams 1" "--batch 32 --streams 4" "--batch 64 --streams 2" "--batch 64 --streams 4" "--batch 48 --streams 3" "--batch 96 --streams 3" "--batch 16 --streams 2"; do run "$a"; done
