# compute-sanitizer over the CUDA paths: memcheck / racecheck / synccheck on one
# N=2^16 HMult+HRot+rescale (every fused kernel), memcheck on the small parity
# tests, the smoke and the peer-exchange shards, racecheck on the NTT passes
for t in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $t --print-limit 10 python tools/sanitize_mech.py 2>&1 | tail -2; done
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_crypt.py tests/test_gpu_encode.py -x -q -m gpu -k "1024 or fixture or small or 256 or 512" 2>&1 | tail -2
SMOKE=1 timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python __graft_entry__.py 2>&1 | tail -2
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/prof_ntt.py 16 1 2>&1 | tail -1
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_limb.py -x -q -m gpu -k "small and True" 2>&1 | tail -2
