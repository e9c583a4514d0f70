"""Whole batched step (B HMult + B HRot over S streams, as bench.py's headline)
eager vs captured once as a CUDA graph and replayed: ops/s and bit equality."""
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_13055_b200 import ckks, dp  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 48
S = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N, L, A, DB, LV = 1 << 16, 24, 8, 55, 24
dev = torch.device("cuda", 0)
C = ckks.CkksContext(ckks.CkksParams(n=N, l=L, alpha=A, delta_bits=DB))
q = torch.tensor(C.primes.astype(np.int64), device=dev)


def rows(prefix, idx):
    u = torch.randint(0, 1 << 62, (*prefix, len(idx), N), device=dev, dtype=torch.int64)
    return (u % q[idx].view(*([1] * len(prefix)), -1, 1)).to(torch.int32).contiguous()


full = list(range(L + A))
D = C.num_digits(L)
relin = ckks.EvaluationKey(rows((D, 2), full))
rot = ckks.EvaluationKey(rows((D, 2), full), ckks.ROTATION, 1)
s = Fraction(1 << DB)
X = ckks.Ciphertext(rows((B, 2), list(range(LV))), s, LV)
Y = ckks.Ciphertext(rows((B, 2), list(range(LV))), s, LV)
subs = [dp.shard_bounds(B, S, i) for i in range(S)]
st = torch.cuda.Stream(dev)
streams = [st] + [torch.cuda.Stream(dev) for _ in range(S - 1)]
o1 = [torch.empty((hi - lo, 2, LV - 2, N), dtype=torch.int32, device=dev) for lo, hi in subs]
o2 = [torch.empty((hi - lo, 2, LV, N), dtype=torch.int32, device=dev) for lo, hi in subs]


def step():
    start = torch.cuda.Event()
    start.record(st)
    done = []
    for k, ((lo, hi), s_k) in enumerate(zip(subs, streams)):
        s_k.wait_event(start)
        with torch.cuda.stream(s_k):
            Xs = ckks.Ciphertext(X.data[lo:hi], s, LV)
            Ys = ckks.Ciphertext(Y.data[lo:hi], s, LV)
            ckks.hmult(C, Xs, Ys, relin, out=o1[k])
            ckks.hrot(C, Xs, 1, rot, out=o2[k])
            e = torch.cuda.Event()
            e.record(s_k)
            done.append(e)
    for e in done:
        st.wait_event(e)


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


with torch.cuda.stream(st):
    ms_e = timed(step)
    ref1 = [t.clone() for t in o1]
    ref2 = [t.clone() for t in o2]
    g = torch.cuda.CUDAGraph()
    st.synchronize()
    with torch.cuda.graph(g, stream=st):
        step()
    for t in o1 + o2:
        t.zero_()
    ms_g = timed(g.replay)
    same = all(torch.equal(a, b) for a, b in zip(ref1 + ref2, o1 + o2))
print(f"B={B} S={S}: eager {ms_e:.3f} ms/step = {2 * B / ms_e * 1e3:.0f} ops/s; graph {ms_g:.3f} ms/step = "
      f"{2 * B / ms_g * 1e3:.0f} ops/s; graph outputs equal eager: {same}")
