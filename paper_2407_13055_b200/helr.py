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
    ip    = sum_{s=1,2,..,F/2} rot_s(ip)            log2(F) HRot + HAdd: slot (i, 0) = <z_i, w>
    ip    = rescale(ip (*) mask)                    PMult, rescale   (-> l-4): keep the (i, 0) slots
    ip    = sum_{s=1,2,..,F/2} rot_{-s}(ip)         log2(F) HRot + HAdd: <z_i, w> in all F slots of i
    x2    = ip * ip                                 HMult            (-> l-6)
    t     = rescale(x2 (*) a3) (+) a1               PMult, rescale, PAdd (-> l-8)
    sig   = t * ip|_(l-8)                           HMult            (-> l-10)
    sig   = sig (+) a0                              PAdd: sig_i = a0 + a1 ip_i + a3 ip_i^3
    g     = sig * Z|_(l-10)                         HMult            (-> l-12)
    g     = sum_{s=F,2F,..,N/4} rot_s(g)            log2(S) HRot + HAdd
    g     = sum over the cts ciphertexts            HAdd tree: slot (i, f) = sum_i' sig_i' z_i'f
    W'    = rescale(W|_(l-12) (*) 1) + rescale(g (*) gamma)   2 PMult, 2 rescale, HAdd (-> l-14)

so W' holds w + gamma * sum_i P(<z_i, w>) z_i in every sample's slots: one
gradient step of logistic regression with the degree-3 polynomial P
(HELR: z_i = y_i (1, x_i), P(t) ~ sigmoid(-t)); tests/test_gpu_helr.py
checks the decrypted W' against the same step in numpy.

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

    def replicate_rotations(self) -> List[int]:
        return [-r for r in self.feature_rotations()]

    def rotations(self) -> List[int]:
        return self.feature_rotations() + self.replicate_rotations() + self.sample_rotations()


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

    `consts` maps 'mask', 'a3', 'a1', 'a0', 'gamma', 'one' to a callable (level, scale) ->
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
        return 14

    def step(self, Z: ckks.Ciphertext, W: ckks.Ciphertext) -> ckks.Ciphertext:
        C, sh = self.ctx, self.shape
        if not Z.batched or Z.batch != sh.cts:
            raise ValueError("Z must be a batch of `cts` ciphertexts")
        if W.batched:
            raise ValueError("W is one ciphertext")
        if Z.level != W.level or Z.level < 16:
            raise ValueError("Z and W must share a level >= 16")
        l = Z.level
        D = self.ctx.default_scale()
        Wb = ckks.Ciphertext(W.data.unsqueeze(0).expand(sh.cts, *W.data.shape).contiguous(), W.scale, l)
        ip = ckks.hmult(C, Z, Wb, self.relin)                                     # l-2
        ip = rotsum(C, ip, sh.feature_rotations(), self.keys)
        ip = ckks.rescale(C, ckks.pmult(C, ip, self._pt("mask", ip.level, D)))     # l-4
        ip = rotsum(C, ip, sh.replicate_rotations(), self.keys)
        x2 = ckks.hmult(C, ip, ip, self.relin)                                    # l-6
        t = ckks.rescale(C, ckks.pmult(C, x2, self._pt("a3", x2.level, D)))       # l-8
        t = ckks.padd(C, t, self._pt("a1", t.level, t.scale))
        sig = ckks.hmult(C, t, drop(ip, t.level), self.relin)                     # l-10
        sig = ckks.padd(C, sig, self._pt("a0", sig.level, sig.scale))
        g = ckks.hmult(C, sig, drop(Z, sig.level), self.relin)                    # l-12
        g = rotsum(C, g, sh.sample_rotations(), self.keys)
        g = batch_sum(C, g)
        # W' = W * 1 + g * gamma: both products rescaled to the common scale
        # g.scale * Delta / qq, so the final HAdd meets the exact-scale check with
        # every plaintext scale <= 2^60 (encode's range, ckks.cpp:284-285)
        upd = ckks.rescale(C, ckks.pmult(C, g, self._pt("gamma", g.level, D)))   # l-14
        wl = ckks.rescale(C, ckks.pmult(C, drop(W, g.level), self._pt("one", g.level, g.scale * D / W.scale)))
        return ckks.hadd(C, wl, upd)

    def op_profile(self) -> Dict[str, int]:
        """Mechanism calls per iteration (each batched over `cts` where it applies)."""
        sh = self.shape
        return {"hmult": 4, "hrot": len(sh.rotations()), "pmult": 4, "rescale": 4, "padd": 2,
                "hadd": len(sh.rotations()) + (sh.cts - 1).bit_length() + 1}
