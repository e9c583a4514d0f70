"""One HMult+relin and one HRot at N=2^16, l=24 (B=2) through every fused
N=2^16 kernel (column / row passes, row pass + KeyMult, fused combine, BConv,
tensor, HRot tail), plus rescale -- small enough to run under
compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
from fractions import Fraction
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_13055_b200 import ckks  # noqa: E402


def main():
    n, l, a, B = 1 << 16, 24, 8, 2
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=55))
    q = torch.tensor(C.primes.astype("int64"), device="cuda")
    D = C.num_digits(l)

    def rows(prefix, idx):
        u = torch.randint(0, 1 << 62, (*prefix, len(idx), n), device="cuda", dtype=torch.int64)
        return (u % q[idx].view(*([1] * len(prefix)), -1, 1)).to(torch.int32).contiguous()

    full = torch.cat([torch.arange(l), l + torch.arange(a)]).cuda()
    evk = ckks.EvaluationKey(rows((D, 2), full))
    rot = ckks.EvaluationKey(rows((D, 2), full), ckks.ROTATION, 1)
    s = Fraction(1 << 55)
    X = ckks.Ciphertext(rows((B, 2), torch.arange(l).cuda()), s, l)
    Y = ckks.Ciphertext(rows((B, 2), torch.arange(l).cuda()), s, l)
    ckks.hmult(C, X, Y, evk)
    ckks.hrot(C, X, 1, rot)
    ckks.rescale(C, X)
    torch.cuda.synchronize()
    print("sanitize_mech ok")


if __name__ == "__main__":
    main()
