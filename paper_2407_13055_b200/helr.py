"""HELR-style logistic-regression iteration (BASELINE.json configs[4]).

The reference implements no bootstrapping, so config 5 is the
HELR-style training iteration of Cheddar's evaluation (after
Han et al., AAAI'19) built ONLY from the evaluator API this package mirrors
(ckks.hpp:170-208): HMult+relinearize (merged rescale), HRot, PMult, PAdd,
HAdd and rescale.  It is a workload driver over the hot path, not new
arithmetic: every output is bit-identical to running the same op sequence
through the reference (tests/test_gpu_helr.py checks it against the C
restatement op by op).

Packing (one mini-batch, `cts` ciphertexts, N/2 slots each): slot
s = sample * F + feature, F = `features` (power of two), S = N/2 / F samples
per ciphertext.  The weight ciphertext W holds the model replicated per
sample.  One iteration (gradient step with a degree-3 sigmoid):

    ip    = Z * W                                  HMult            (l -> l-2)
    ip    = sum_{s=1,2,..,F/2} rot_s(ip)            log2(F) HRot + HAdd
    x2    = ip * ip                                 HMult            (-> l-4)
    t     = rescale(x2 (*) a3) (+) a1               PMult, rescale, PAdd (-> l-6)
    sig   = t * ip|_(l-6)                           HMult            (-> l-8)
    sig   = sig (+) a0                              PAdd
    g     = sig * Z|_(l-8)                          HMult            (-> l-10)
    g     = sum_{s=F,2F,..,N/4} rot_s(g)            log2(S) HRot + HAdd
    g     = sum over the cts ciphertexts            HAdd tree
    W'    = W|_(l-12) (+) rescale(g (*) gamma)      PMult, rescale, HAdd (-> l-12)

`x|_m` keeps the first m RNS rows (a ciphertext mod Q_l is one mod Q_m).
The ciphertexts of a mini-batch are processed as ONE batched ciphertext, so
every mechanism above is one batched launch sequence with the key read once.
Plaintext constants are supplied by the caller (encoding is host-side in the
reference); their scales are chosen so that every HAdd / PAdd meets the
reference's scale check exactly.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Dict, List

import torch

from . import ckks


@dataclass
class HelrShape:
    n: int = 1 << 16
    features: int = 256  # F (power of two)
    cts: int = 8         # ciphertexts per mini-batch

    @property
    def slots(self) -> int:
        return self.n // 2

    @property
    def samples_per_ct(self) -> int:
        return self.slots // self.features

    def feature_rotations(self) -> List[int]:
        return [1 << k for k in range(self.features.bit_length() - 1)]

    def sample_rotations(self) -> List[int]:
        out, s = [], self.features
        while s < self.slots:
            out.append(s)
            s <<= 1
        return out

    def rotations(self) -> List[int]:
        return self.feature_rotations() + self.sample_rotations()


def drop(ct: ckks.Ciphertext, level: int) -> ckks.Ciphertext:
    """Keep the first `level` RNS rows (modulus switch down by dropping limbs)."""
    if level > ct.level:
        raise ValueError("cannot raise the level")
    return ckks.Ciphertext(ct.data[..., :level, :].contiguous(), ct.scale, level, ct.pending_rescale)


def rotsum(ctx: ckks.CkksContext, ct: ckks.Ciphertext, steps: List[int], keys: Dict[int, ckks.EvaluationKey]):
    for r in steps:
        ct = ckks.hadd(ctx, ct, ckks.hrot(ctx, ct, r, keys[r]))
    return ct


def batch_sum(ctx: ckks.CkksContext, ct: ckks.Ciphertext) -> ckks.Ciphertext:
    """HAdd tree over the leading batch dimension -> one ciphertext."""
    data = ct.data
    while data.shape[0] > 1:
        h = data.shape[0] // 2
        s = ckks.hadd(ctx, ckks.Ciphertext(data[:h].contiguous(), ct.scale, ct.level),
                      ckks.Ciphertext(data[h:2 * h].contiguous(), ct.scale, ct.level)).data
        if data.shape[0] % 2:
            s = torch.cat([s, data[2 * h:]], 0)
        data = s
    return ckks.Ciphertext(data[0], ct.scale, ct.level)


class HelrIteration:
    """One HELR-style gradient step over a mini-batch of encrypted samples.

    `consts` maps 'a3', 'a1', 'a0', 'gamma' to a callable (level, scale) ->
    Plaintext (evaluation domain, Montgomery, Q-prefix rows): the caller's
    encoder.  The scales requested here make every addition exact-scale."""

    def __init__(self, ctx: ckks.CkksContext, shape: HelrShape, relin: ckks.EvaluationKey,
                 rot_keys: Dict[int, ckks.EvaluationKey], consts):
        missing = [r for r in shape.rotations() if r not in rot_keys]
        if missing:
            raise ValueError(f"missing rotation keys {missing}")
        if shape.n != ctx.n:
            raise ValueError("ring dimension mismatch")
        self.ctx, self.shape, self.relin, self.keys, self.consts = ctx, shape, relin, rot_keys, consts
        self._pt_cache = {}

    def _pt(self, name: str, level: int, scale: Fraction) -> ckks.Plaintext:
        key = (name, level, scale)
        if key not in self._pt_cache:
            self._pt_cache[key] = self.consts[name](level, scale)
        return self._pt_cache[key]

    def levels_used(self) -> int:
        return 12

    def step(self, Z: ckks.Ciphertext, W: ckks.Ciphertext) -> ckks.Ciphertext:
        C, sh = self.ctx, self.shape
        if not Z.batched or Z.batch != sh.cts:
            raise ValueError("Z must be a batch of `cts` ciphertexts")
        if W.batched:
            raise ValueError("W is one ciphertext")
        if Z.level != W.level or Z.level < 14:
            raise ValueError("Z and W must share a level >= 14")
        l = Z.level
        Wb = ckks.Ciphertext(W.data.unsqueeze(0).expand(sh.cts, *W.data.shape).contiguous(), W.scale, l)
        ip = ckks.hmult(C, Z, Wb, self.relin)                                     # l-2
        ip = rotsum(C, ip, sh.feature_rotations(), self.keys)
        x2 = ckks.hmult(C, ip, ip, self.relin)                                    # l-4
        t = ckks.pmult(C, x2, self._pt("a3", x2.level, self.ctx.default_scale()))
        t = ckks.rescale(C, t)                                                    # l-6
        t = ckks.padd(C, t, self._pt("a1", t.level, t.scale))
        sig = ckks.hmult(C, t, drop(ip, t.level), self.relin)                     # l-8
        sig = ckks.padd(C, sig, self._pt("a0", sig.level, sig.scale))
        g = ckks.hmult(C, sig, drop(Z, sig.level), self.relin)                    # l-10
        g = rotsum(C, g, sh.sample_rotations(), self.keys)
        g = batch_sum(C, g)
        # W' = W + gamma * g with the plaintext scale chosen so the sum is exact-scale
        lo = g.level - 2
        qq = int(C.q_primes[g.level - 2]) * int(C.q_primes[g.level - 1])
        upd = ckks.pmult(C, g, self._pt("gamma", g.level, W.scale * qq / g.scale))
        upd = ckks.rescale(C, upd)                                                # l-12
        return ckks.hadd(C, drop(W, lo), upd)

    def op_profile(self) -> Dict[str, int]:
        """Mechanism calls per iteration (each batched over `cts` where it applies)."""
        sh = self.shape
        return {"hmult": 4, "hrot": len(sh.rotations()), "pmult": 2, "rescale": 2, "padd": 2,
                "hadd": len(sh.rotations()) + (sh.cts - 1).bit_length() + 1}
