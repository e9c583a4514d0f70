# persistent-grid caps (CTAs per SM) for the 2-stream overlap: single-factor sweeps
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-small --no-sweep --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['bit_exact'])"; }
run X=0
for c in 4 3; do run CK32_COL_CTAS=$c; done
for c in 4 3 2; do run CK32_ROW_CTAS=$c; done
for c in 6 4; do run CK32_KM_CTAS=$c; done
for c in 3 2; do run CK32_BCONV_CTAS=$c; done
run "CK32_COL_CTAS=4 CK32_KM_CTAS=6"
run "CK32_COL_CTAS=4 CK32_ROW_CTAS=3 CK32_KM_CTAS=6"
run X=0
