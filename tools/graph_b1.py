"""Small-batch latency: eager C-ABI calls vs the same HMult+HRot sequence
captured once in a CUDA graph (torch.cuda.CUDAGraph) and replayed.
    python tools/graph_b1.py [batch] [reps]"""
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_13055_b200 import ckks  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    n, l, a = 1 << 16, 24, 8
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=55))
    q = torch.tensor(C.primes.astype(np.int64), device="cuda")

    def rows(prefix, idx):
        u = torch.randint(0, 1 << 62, (*prefix, len(idx), n), device="cuda", dtype=torch.int64)
        return (u % q[idx].view(*([1] * len(prefix)), -1, 1)).to(torch.int32).contiguous()

    full = torch.cat([torch.arange(l), l + torch.arange(a)]).cuda()
    relin = ckks.EvaluationKey(rows((3, 2), full))
    rot = ckks.EvaluationKey(rows((3, 2), full), ckks.ROTATION, 1)
    s = Fraction(1 << 55)
    X = ckks.Ciphertext(rows((B, 2), torch.arange(l).cuda()), s, l)
    Y = ckks.Ciphertext(rows((B, 2), torch.arange(l).cuda()), s, l)
    st = torch.cuda.Stream()
    outs = {}
    with torch.cuda.stream(st):
        def step():
            outs["m"] = ckks.hmult(C, X, Y, relin)
            outs["r"] = ckks.hrot(C, X, 1, rot)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            step()
        e1.record(st)
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / reps
        ref_m, ref_r = outs["m"].data.clone(), outs["r"].data.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            step()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(outs["m"].data, ref_m) and torch.equal(outs["r"].data, ref_r)
        e0.record(st)
        for _ in range(reps):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        graph = e0.elapsed_time(e1) / reps
        # HMult and HRot on two forked streams inside one captured graph
        s2 = torch.cuda.Stream()

        def step2():
            s2.wait_stream(st)
            outs["m"] = ckks.hmult(C, X, Y, relin)
            with torch.cuda.stream(s2):
                outs["r"] = ckks.hrot(C, X, 1, rot)
            st.wait_stream(s2)
        for _ in range(3):
            step2()
        torch.cuda.synchronize()
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=st):
            step2()
        g2.replay()
        torch.cuda.synchronize()
        assert torch.equal(outs["m"].data, ref_m) and torch.equal(outs["r"].data, ref_r)
        e0.record(st)
        for _ in range(reps):
            g2.replay()
        e1.record(st)
        torch.cuda.synchronize()
        graph2 = e0.elapsed_time(e1) / reps
    print(f"B={B}: graph on 2 streams {graph2 * 1e3:.1f} us ({2 * B / graph2 * 1e3:.0f} ops/s)")
    print(f"B={B}: eager {eager * 1e3:.1f} us per HMult+HRot ({2 * B / eager * 1e3:.0f} ops/s), "
          f"graph {graph * 1e3:.1f} us ({2 * B / graph * 1e3:.0f} ops/s), bit-exact replay")


if __name__ == "__main__":
    main()
