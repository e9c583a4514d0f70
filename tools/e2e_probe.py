"""Repeatability probe of bench.py's e2e leg: the same HostPipeline workload
timed several times in one process, with the caching allocator's cudaMalloc /
retry counters between repeats (looking for allocator or arena churn)."""
import sys, time
from fractions import Fraction
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_13055_b200 import ckks
from paper_2407_13055_b200.pipeline import HostPipeline

N, L, A, DB, LV, B = 1 << 16, 24, 8, 55, 24, 32
chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 4
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
depth = int(sys.argv[3]) if len(sys.argv) > 3 else 2
pipe = HostPipeline(dev, chunk=chunk, depth=depth)
inplace = len(sys.argv) > 2 and sys.argv[2] == "inplace"
def fn(d, o=None):
    cx = ckks.Ciphertext(d[0], s, LV)
    return (ckks.hmult(C, cx, ckks.Ciphertext(d[1], s, LV), relin, out=o[0] if o else None).data,
            ckks.hrot(C, cx, 1, rot, out=o[1] if o else None).data)
st = torch.cuda.current_stream(dev)
for _ in range(3): pipe.run([hx, hy], fn, [ho1, ho2], outputs_in_place=inplace)
torch.cuda.synchronize()
for rep in range(6):
    m0 = torch.cuda.memory_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record(st)
    for _ in range(10): last = pipe.run([hx, hy], fn, [ho1, ho2], outputs_in_place=inplace)
    st.wait_event(last); b.record(st); torch.cuda.synchronize()
    ms = a.elapsed_time(b); m1 = torch.cuda.memory_stats()
    print(f"chunk {chunk} depth {depth} inplace {inplace} rep {rep}: {2 * B * 10 / (ms / 1e3):.0f} ops/s  host {1e3 * (time.perf_counter() - t0):.0f} ms  "
          f"cudaMalloc +{m1.get('num_device_alloc', 0) - m0.get('num_device_alloc', 0)} retries +{m1.get('num_alloc_retries', 0) - m0.get('num_alloc_retries', 0)}")
