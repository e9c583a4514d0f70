# round-2: full GPU suite + compute-sanitizer over the round-2 kernels (TMA column pass,
# k_row_keymult8, L2-prefetch combine, galois automorphism, element-wise, device-epoch peer exchange)
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -q -m gpu 2>&1 | tail -3
for t in memcheck racecheck synccheck; do echo "== $t mech"; timeout 900 compute-sanitizer --tool $t --print-limit 10 python tools/sanitize_mech.py 2>&1 | tail -2; done
echo "== memcheck small parity incl. new ABI"; timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "elementwise or automorphism_both or wire or 1024" 2>&1 | tail -2
echo "== racecheck ntt"; timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/prof_ntt.py 16 1 2>&1 | tail -1
echo "== memcheck limb"; timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_limb.py -x -q -m gpu -k "small or rejects" 2>&1 | tail -2
