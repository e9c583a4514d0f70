"""Standalone driver for profiling the NTT / INTT kernels (ncu target).

    [LOGN=17] python tools/prof_ntt.py [rows] [reps]

Transforms `rows` limbs (cycling over the 32 primes of config 1) in one
batched launch pair, `reps` times, and prints the CUDA-event time per limb.
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_13055_b200 import ckks  # noqa: E402


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 768
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    import os
    n, l, a = 1 << int(os.environ.get("LOGN", "16")), 24, 8
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=55))
    g = np.array([i % (l + a) for i in range(rows)], np.uint32)
    q = torch.tensor(C.primes[g].astype(np.int64), device="cuda")
    x = (torch.randint(0, 1 << 62, (rows, n), device="cuda", dtype=torch.int64) % q[:, None]).to(torch.int32)
    from paper_2407_13055_b200 import _native as nat

    garr = nat.u32_array(g)
    st = C.stream()
    for kind in ("fwd", "inv"):
        fn = (lambda: nat.call("ck_ntt_forward", C.handle, x.data_ptr(), rows, garr, st)) if kind == "fwd" else \
             (lambda: nat.call("ck_intt_inverse", C.handle, x.data_ptr(), rows, garr, None, st))
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        ns_limb = ms * 1e6 / rows
        gbs = rows * 8 * n / (ms * 1e6)
        print(f"{kind}: {ms:.3f} ms for {rows} limbs = {ns_limb:.1f} ns/limb, {gbs:.0f} GB/s algorithmic "
              f"({gbs / 6550.1:.3f} of measured HBM)")


if __name__ == "__main__":
    main()
