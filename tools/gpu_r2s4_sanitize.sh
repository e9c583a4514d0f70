# compute-sanitizer over the session-4 kernel changes (grouped-GS inverse column pass, keymult8 twiddles by
# cp.async) through one HMult + HRot + rescale (every fused kernel), plus the NTT passes alone
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do echo "== $t mech"; timeout 900 compute-sanitizer --tool $t --print-limit 10 python tools/sanitize_mech.py 2>&1 | tail -2; done
for t in memcheck racecheck; do echo "== $t ntt"; timeout 900 compute-sanitizer --tool $t --print-limit 10 python tools/prof_ntt.py 16 1 2>&1 | tail -1; done
