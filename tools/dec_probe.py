import sys, numpy as np, torch
sys.path[:0] = ['/root/repo', '/root/repo/oracle']
from fractions import Fraction
from paper_2407_13055_b200 import ckks
from pyoracle import Reference
ref = Reference()
for (n, l, a, level) in [(1024, 8, 3, 8), (65536, 24, 8, 24), (65536, 24, 8, 3)]:
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=55))
    r = np.random.default_rng(7 + n).uniform(-1.0, 1.0, (n // 2, 2)); z = r[:, 0] + 1j * r[:, 1]
    for num, den in [(1 << 55, 1), (3 << 53, 5), ((1 << 60) - 1, 3)]:
        rows = ref.encode(n, l, a, 55, z, num, den, level)
        want = ref.decode(n, l, a, 55, rows, level, num, den)
        pt = ckks.Plaintext(ckks.Polynomial(torch.from_numpy(rows.astype(np.int64).astype(np.int32)).cuda(), level, 0), Fraction(num, den), level)
        got = ckks.decode(C, pt)
        d = np.abs(got - want)
        print(n, level, num, den, 'max diff', d.max(), 'n differing', int((got != want).sum()), 'of', got.size)
