"""e2e pipeline vs the PCIe link: the bench's HostPipeline step (B = 32 HMult + HRot,
chunks of 4) timed (a) as is, (b) with the evaluator calls replaced by nothing
(copies only, same chunking), (c) the step's bytes as two big concurrent copies."""
import sys, time
from fractions import Fraction
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_13055_b200 import ckks
from paper_2407_13055_b200.pipeline import HostPipeline

N, L, A, DB, LV, B = 1 << 16, 24, 8, 55, 24, 32
dev = torch.device("cuda", 0)
C = ckks.CkksContext(ckks.CkksParams(n=N, l=L, alpha=A, delta_bits=DB))
q = torch.tensor(C.primes.astype(np.int64), device=dev)
def rows(prefix, idx):
    u = torch.randint(0, 1 << 62, (*prefix, len(idx), N), device=dev, dtype=torch.int64)
    return (u % q[idx].view(*([1] * len(prefix)), -1, 1)).to(torch.int32).contiguous()
full = list(range(L + A)); D = C.num_digits(L)
relin = ckks.EvaluationKey(rows((D, 2), full)); rot = ckks.EvaluationKey(rows((D, 2), full), ckks.ROTATION, 1)
s = Fraction(1 << DB)
hx = rows((B, 2), list(range(LV))).cpu().pin_memory(); hy = rows((B, 2), list(range(LV))).cpu().pin_memory()
ho1 = torch.empty((B, 2, LV - 2, N), dtype=torch.int32).pin_memory(); ho2 = torch.empty((B, 2, LV, N), dtype=torch.int32).pin_memory()
st = torch.cuda.current_stream(dev)
def timed(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): last = fn()
    if last is not None: st.wait_event(last)
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for chunk, depth in ((4, 2), (8, 2), (16, 2), (2, 3)):
    pipe = HostPipeline(dev, chunk=chunk, depth=depth)
    def fn_full(d, o):
        cx = ckks.Ciphertext(d[0], s, LV)
        return (ckks.hmult(C, cx, ckks.Ciphertext(d[1], s, LV), relin, out=o[0]).data, ckks.hrot(C, cx, 1, rot, out=o[1]).data)
    def fn_copy(d, o):
        return o[0], o[1]
    ms_full = timed(lambda: pipe.run([hx, hy], fn_full, [ho1, ho2], outputs_in_place=True))
    ms_copy = timed(lambda: pipe.run([hx, hy], fn_copy, [ho1, ho2], outputs_in_place=True))
    print(f"chunk {chunk} depth {depth}: full {ms_full:.2f} ms/step ({2 * B / ms_full * 1e3:.0f} ops/s), copies only {ms_copy:.2f} ms/step")
din = [torch.empty_like(hx, device=dev), torch.empty_like(hy, device=dev)]
dout = [torch.empty_like(ho1, device=dev), torch.empty_like(ho2, device=dev)]
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
def big():
    ev = torch.cuda.Event(); ev.record(st); s1.wait_event(ev); s2.wait_event(ev)
    with torch.cuda.stream(s1):
        for d_, h_ in zip(din, (hx, hy)): d_.copy_(h_, non_blocking=True)
    with torch.cuda.stream(s2):
        for h_, d_ in zip((ho1, ho2), dout): h_.copy_(d_, non_blocking=True)
    st.wait_stream(s1); st.wait_stream(s2)
    return None
print(f"two big concurrent copies: {timed(big, 5):.2f} ms/step")
