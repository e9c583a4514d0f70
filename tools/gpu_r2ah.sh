# NTT per-limb time vs working-set size: L2-resident (96-384 limbs = 25-100 MB) vs HBM-streaming (768-3072)
for r in 96 192 384 768 1536 3072; do echo "rows=$r"; timeout 120 python tools/prof_ntt.py $r 20; done
