"""Python mirror of the reference evaluator API (ckks.hpp:102-219) over the
B200 C-ABI (include/ck32_b200.h).

Names, argument meaning, level/scale ledger and error behaviour follow the
reference: ``std::invalid_argument`` becomes ``ValueError``.  Residues live on
the GPU as int32 tensors holding canonical values in [0, q) (bit-identical to
the reference's ``correct_lazy`` view); every compute call goes through the
native library — there is no host fallback.

Batching: any Ciphertext may carry a leading batch dimension
(``data`` of shape ``[B, 2, level, n]``); hmult / hrot / rescale / hadd /
padd / pmult process the whole batch in one launch sequence with the key
streamed once.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from fractions import Fraction
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native as nat

COEFFICIENT, EVALUATION = "coefficient", "evaluation"
RELIN, ROTATION = "relin", "rotation"
COUNTER_NAMES = ("modup", "moddown", "ntt", "intt", "keymult", "bconv", "rescale")  # ckks.hpp:34-44


@dataclass
class CkksParams:
    """ckks.hpp:46-54 (hamming / sigma only matter for host-side key sampling)."""
    n: int = 1 << 16
    l: int = 54
    alpha: int = 14
    delta_bits: int = 48
    hamming: int = 256
    sigma: float = 3.2
    lazy_rescale: bool = False


def _ptr(t: torch.Tensor) -> int:
    if not t.is_cuda:
        raise ValueError("tensor must live on the GPU")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


class CkksContext:
    """CkksContext (ckks.cpp:160-176): basis, twiddles and per-level tables
    on one device."""

    def __init__(self, params: CkksParams, device: int = 0, primes: Optional[Sequence[int]] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("ck32-b200 needs a CUDA device (no CPU fallback)")
        self.params = params
        self.device = torch.device("cuda", device)
        p = nat.ck_params(params.n, params.l, params.alpha, params.delta_bits, int(params.lazy_rescale))
        h = ctypes.c_void_p()
        arr = nat.u32_array(primes) if primes is not None else None
        with torch.cuda.device(self.device):
            nat.call("ck_context_create", ctypes.byref(p), arr, device, ctypes.byref(h))
        self._h = h
        out = (ctypes.c_uint32 * (params.l + params.alpha))()
        nat.call("ck_context_primes", h, out)
        self.primes = np.array(list(out), dtype=np.uint32)
        self.q_primes = self.primes[: params.l]
        self.p_primes = self.primes[params.l:]

    # ---------------------------------------------------------------- misc --
    @property
    def handle(self):
        return self._h

    @property
    def n(self) -> int:
        return self.params.n

    @property
    def slots(self) -> int:
        return self.params.n // 2

    def num_digits(self, level: int) -> int:
        return (level + self.params.alpha - 1) // self.params.alpha

    def default_scale(self) -> Fraction:
        return Fraction(1 << self.params.delta_bits)

    def stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def counters(self) -> dict:
        out = (ctypes.c_uint64 * 7)()
        nat.call("ck_context_counters", self._h, out)
        return dict(zip(COUNTER_NAMES, list(out)))

    def reset_counters(self) -> None:
        nat.call("ck_context_reset_counters", self._h)

    def profile(self, enable: bool = True) -> None:
        """Start (clear) / stop per-kernel-class CUDA-event timing."""
        nat.call("ck_profile", self._h, int(enable))

    def profile_read(self) -> List[dict]:
        buf = (nat.ck_prof_stat * 16)()
        cnt = ctypes.c_uint32()
        nat.call("ck_profile_read", self._h, buf, 16, ctypes.byref(cnt))
        return [{"name": s.name.decode(), "groups": s.groups, "launches": s.launches, "ms": s.ms, "bytes": s.bytes}
                for s in buf[: cnt.value]]

    def launch_count(self) -> int:
        return int(nat.lib().ck_launch_count(self._h))

    def gidx(self, level: int, p_rows: int = 0) -> np.ndarray:
        return np.concatenate([np.arange(level), self.params.l + np.arange(p_rows)]).astype(np.uint32)

    def empty(self, *shape) -> torch.Tensor:
        return torch.empty(shape, dtype=torch.int32, device=self.device)

    def close(self):
        if getattr(self, "_h", None):
            torch.cuda.synchronize(self.device)
            nat.call("ck_context_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------- types --
@dataclass
class Polynomial:
    """poly.hpp:74-119: rows x n residues, Q-prefix rows then P rows."""
    data: torch.Tensor
    q_count: int
    p_count: int = 0
    domain: str = EVALUATION
    mont: bool = True

    @property
    def rows(self) -> int:
        return self.q_count + self.p_count

    def clone(self) -> "Polynomial":
        return Polynomial(self.data.clone(), self.q_count, self.p_count, self.domain, self.mont)


@dataclass
class Plaintext:
    poly: Polynomial
    scale: Fraction
    level: int


@dataclass
class Ciphertext:
    """ckks.hpp:61-66; data is [2, level, n] (b, a) or [B, 2, level, n]."""
    data: torch.Tensor
    scale: Fraction
    level: int
    pending_rescale: bool = False

    @property
    def batched(self) -> bool:
        return self.data.dim() == 4

    @property
    def batch(self) -> int:
        return self.data.shape[0] if self.batched else 1

    @property
    def b(self) -> torch.Tensor:
        return self.data[..., 0, :, :]

    @property
    def a(self) -> torch.Tensor:
        return self.data[..., 1, :, :]


@dataclass
class EvaluationKey:
    """ckks.hpp:79-84; data is [D, 2, L+alpha, n] over the full PQ basis."""
    data: torch.Tensor
    kind: str = RELIN
    rotation: int = 0


@dataclass
class HoistState:
    """ckks.hpp:88-91: D ModUp-extended digits over (level + alpha) rows."""
    level: int
    digits: torch.Tensor  # [D, level + alpha, n]


# ------------------------------------------------------------------ checks --
def _check_pair(ctx: CkksContext, ct: Ciphertext) -> None:  # ckks.cpp:122-129
    shape = ct.data.shape[-3:]
    if tuple(shape) != (2, ct.level, ctx.n):
        raise ValueError("ciphertext level/shape mismatch")
    if ct.level < 1 or ct.level > ctx.params.l:
        raise ValueError("ciphertext level/shape mismatch")


def _check_same_scale(a: Fraction, b: Fraction) -> None:  # ckks.cpp:131-136
    if abs(a - b) * (1 << 40) > a:
        raise ValueError("scale mismatch beyond tolerance")


def _check_eval_mont(p: Polynomial, what: str) -> None:  # ckks.cpp:115-120
    if p.domain != EVALUATION or not p.mont:
        raise ValueError(f"{what}: expected evaluation-domain Montgomery form")


def _flushed(ctx: CkksContext, ct: Ciphertext) -> Ciphertext:  # ckks.cpp:664-676
    return rescale(ctx, ct) if ct.pending_rescale else ct


def _qq(ctx: CkksContext, level: int) -> int:
    return int(ctx.q_primes[level - 2]) * int(ctx.q_primes[level - 1])


# ------------------------------------------------------- element-wise ops --
def hadd(ctx: CkksContext, x: Ciphertext, y: Ciphertext) -> Ciphertext:  # ckks.cpp:557-571
    _check_pair(ctx, x)
    _check_pair(ctx, y)
    if x.level != y.level:
        raise ValueError("level mismatch")
    if x.pending_rescale != y.pending_rescale:
        raise ValueError("pending-rescale state mismatch")
    _check_same_scale(x.scale, y.scale)
    if x.data.shape != y.data.shape:
        raise ValueError("batch mismatch")
    out = torch.empty_like(x.data)
    nat.call("ck_hadd", ctx.handle, x.level, x.batch, _ptr(x.data), _ptr(y.data), _ptr(out), ctx.stream())
    return Ciphertext(out, x.scale, x.level, x.pending_rescale)


def _pt_check(ctx, ct, pt, what):
    _check_pair(ctx, ct)
    _check_eval_mont(pt.poly, what)
    if ct.level != pt.level or pt.poly.p_count != 0:
        raise ValueError("level mismatch")


def padd(ctx: CkksContext, ct: Ciphertext, pt: Plaintext) -> Ciphertext:  # ckks.cpp:573-584
    _pt_check(ctx, ct, pt, "padd")
    _check_same_scale(ct.scale, pt.scale)
    out = torch.empty_like(ct.data)
    nat.call("ck_padd", ctx.handle, ct.level, ct.batch, _ptr(ct.data), _ptr(pt.poly.data), _ptr(out), ctx.stream())
    return Ciphertext(out, ct.scale, ct.level, ct.pending_rescale)


def pmult(ctx: CkksContext, ct: Ciphertext, pt: Plaintext) -> Ciphertext:  # ckks.cpp:586-600
    _pt_check(ctx, ct, pt, "pmult")
    out = torch.empty_like(ct.data)
    nat.call("ck_pmult", ctx.handle, ct.level, ct.batch, _ptr(ct.data), _ptr(pt.poly.data), _ptr(out), ctx.stream())
    return Ciphertext(out, ct.scale * pt.scale, ct.level, ct.pending_rescale)


# ------------------------------------------------------------- mechanisms --
def rescale(ctx: CkksContext, ct: Ciphertext) -> Ciphertext:  # ckks.cpp:789-802
    _check_pair(ctx, ct)
    l = ct.level
    if l < 4:
        raise ValueError("level exhausted")
    shape = list(ct.data.shape)
    shape[-2] = l - 2
    out = torch.empty(shape, dtype=torch.int32, device=ctx.device)
    nat.call("ck_rescale", ctx.handle, l, ct.batch, _ptr(ct.data), _ptr(out), ctx.stream())
    return Ciphertext(out, ct.scale / _qq(ctx, l), l - 2, False)


def mod_up(ctx: CkksContext, d: Polynomial) -> HoistState:  # ckks.cpp:680-731
    _check_eval_mont(d, "mod_up")
    if d.p_count != 0:
        raise ValueError("mod_up input must be Q-only")
    l = d.q_count
    out = ctx.empty(ctx.num_digits(l), l + ctx.params.alpha, ctx.n)
    nat.call("ck_mod_up", ctx.handle, l, _ptr(d.data), _ptr(out), ctx.stream())
    return HoistState(l, out)


def key_mult(ctx: CkksContext, hoist: HoistState, evk: EvaluationKey) -> Tuple[Polynomial, Polynomial]:
    """ckks.cpp:733-770"""
    if evk.data.shape[0] < hoist.digits.shape[0]:
        raise ValueError("evaluation key has too few digits")
    l, a = hoist.level, ctx.params.alpha
    v = ctx.empty(2, l + a, ctx.n)
    nat.call("ck_key_mult", ctx.handle, l, _ptr(hoist.digits), _ptr(evk.data), _ptr(v), ctx.stream())
    return Polynomial(v[0], l, a), Polynomial(v[1], l, a)


def mod_down(ctx: CkksContext, v: Polynomial) -> Polynomial:  # ckks.cpp:772-776
    if v.p_count != ctx.params.alpha:
        raise ValueError("mod_down expects a P-extended polynomial")
    out = ctx.empty(v.q_count, ctx.n)
    nat.call("ck_mod_down", ctx.handle, v.q_count, _ptr(v.data.contiguous()), _ptr(out), ctx.stream())
    return Polynomial(out, v.q_count, 0)


def key_switch(ctx: CkksContext, d: Polynomial, evk: EvaluationKey) -> Tuple[Polynomial, Polynomial]:
    """ckks.cpp:778-787"""
    _check_eval_mont(d, "mod_up")
    if d.p_count != 0:
        raise ValueError("mod_up input must be Q-only")
    l = d.q_count
    out = ctx.empty(2, l, ctx.n)
    nat.call("ck_key_switch", ctx.handle, l, _ptr(d.data), _ptr(evk.data), _ptr(out), ctx.stream())
    return Polynomial(out[0], l), Polynomial(out[1], l)


def _out_tensor(ctx: CkksContext, shape, out: Optional[torch.Tensor]) -> torch.Tensor:
    """The caller's output buffer (checked), or a fresh one.  Passing ``out``
    keeps steady-state serving loops free of allocations (the caching
    allocator's cudaMalloc synchronises the device)."""
    if out is None:
        return torch.empty(shape, dtype=torch.int32, device=ctx.device)
    if tuple(out.shape) != tuple(shape) or out.dtype != torch.int32 or out.device != ctx.device:
        raise ValueError(f"out must be an int32 tensor of shape {tuple(shape)} on {ctx.device}")
    _ptr(out)
    return out


def hmult(ctx: CkksContext, x_in: Ciphertext, y_in: Ciphertext, relin: EvaluationKey,
          out: Optional[torch.Tensor] = None) -> Ciphertext:
    """ckks.cpp:804-865 (merged ModDown+rescale unless params.lazy_rescale)."""
    if relin.kind != RELIN:
        raise ValueError("hmult needs a relinearization key")
    x, y = _flushed(ctx, x_in), _flushed(ctx, y_in)
    _check_pair(ctx, x)
    _check_pair(ctx, y)
    if x.level != y.level:
        raise ValueError("level mismatch")
    l = x.level
    if l < 4:
        raise ValueError("level exhausted")
    if x.data.shape != y.data.shape:
        raise ValueError("batch mismatch")
    lazy = ctx.params.lazy_rescale
    shape = list(x.data.shape)
    shape[-2] = l if lazy else l - 2
    out = _out_tensor(ctx, shape, out)
    nat.call("ck_hmult", ctx.handle, l, x.batch, _ptr(x.data), _ptr(y.data), _ptr(relin.data), _ptr(out),
             ctx.stream())
    if lazy:
        return Ciphertext(out, x.scale * y.scale, l, True)
    return Ciphertext(out, x.scale * y.scale / _qq(ctx, l), l - 2, False)


def hrot(ctx: CkksContext, ct_in: Ciphertext, r: int, evk: EvaluationKey,
         out: Optional[torch.Tensor] = None) -> Ciphertext:  # ckks.cpp:890-897
    ct = _flushed(ctx, ct_in)
    _check_pair(ctx, ct)
    if evk.kind != ROTATION or evk.rotation != r:
        raise ValueError("rotation key mismatch")
    out = _out_tensor(ctx, ct.data.shape, out)
    nat.call("ck_hrot", ctx.handle, ct.level, ct.batch, _ptr(ct.data), int(r), _ptr(evk.data), _ptr(out),
             ctx.stream())
    return Ciphertext(out, ct.scale, ct.level, False)


def hoisted_rotations(ctx: CkksContext, ct_in: Ciphertext, rotations: Sequence[int],
                      evks: Sequence[Optional[EvaluationKey]]) -> List[Ciphertext]:
    """ckks.cpp:899-925: one ModUp shared across rotations."""
    if len(rotations) != len(evks):
        raise ValueError("rotation/key count mismatch")
    ct = _flushed(ctx, ct_in)
    _check_pair(ctx, ct)
    if ct.batched:
        raise ValueError("hoisted rotations take one ciphertext")
    for r, k in zip(rotations, evks):
        if r != 0 and (k is None or k.kind != ROTATION or k.rotation != r):
            raise ValueError("rotation key mismatch")
    cnt = len(rotations)
    out = ctx.empty(cnt, 2, ct.level, ctx.n)
    rots = (ctypes.c_int64 * max(cnt, 1))(*[int(r) for r in rotations])
    keys = (ctypes.c_void_p * max(cnt, 1))(*[(_ptr(k.data) if (k is not None and r != 0) else None)
                                             for r, k in zip(rotations, evks)])
    nat.call("ck_hoisted_rotations", ctx.handle, ct.level, _ptr(ct.data), cnt, rots, keys, _ptr(out), ctx.stream())
    return [Ciphertext(out[i], ct.scale, ct.level, False) for i in range(cnt)]


def hoisted_rotate_accumulate(ctx: CkksContext, ct_in: Ciphertext, rotations: Sequence[int],
                              pts: Sequence[Plaintext], evks: Sequence[Optional[EvaluationKey]]) -> Ciphertext:
    """ckks.cpp:945-1012: sum_k pt_k * rot_k(ct) with one ModUp and one ModDown."""
    if not rotations or len(rotations) != len(pts) or len(rotations) != len(evks):
        raise ValueError("rotation/plaintext/key count mismatch")
    ct = _flushed(ctx, ct_in)
    _check_pair(ctx, ct)
    l, a = ct.level, ctx.params.alpha
    for pt in pts:
        _check_eval_mont(pt.poly, "hoisted accumulate")
        if pt.level != l or pt.poly.p_count != a:
            raise ValueError("plaintexts must be P-extended at the ciphertext level")
        _check_same_scale(pts[0].scale, pt.scale)
    for r, k in zip(rotations, evks):
        if r != 0 and (k is None or k.kind != ROTATION or k.rotation != r):
            raise ValueError("rotation key mismatch")
    cnt = len(rotations)
    out = ctx.empty(2, l, ctx.n)
    rots = (ctypes.c_int64 * cnt)(*[int(r) for r in rotations])
    pp = (ctypes.c_void_p * cnt)(*[_ptr(p.poly.data) for p in pts])
    kp = (ctypes.c_void_p * cnt)(*[(_ptr(k.data) if (k is not None and r != 0) else None)
                                   for r, k in zip(rotations, evks)])
    nat.call("ck_hoisted_rotate_accumulate", ctx.handle, l, _ptr(ct.data), cnt, rots, pp, kp, _ptr(out),
             ctx.stream())
    return Ciphertext(out, ct.scale * pts[0].scale, l, False)


# --------------------------------------------------------------- encoding --
def log2_rational(r: Fraction) -> float:
    """ckks.cpp:140-158, operation for operation (52-bit mantissa window)."""
    num, den = r.numerator, r.denominator
    if num <= 0:
        raise ValueError("log2 of non-positive rational")
    bn, bd = num.bit_length() - 1, den.bit_length() - 1
    shift = 0
    if bn > 52:
        num >>= bn - 52
        shift += bn - 52
    if bd > 52:
        den >>= bd - 52
        shift -= bd - 52
    return float(shift) + math.log2(float(num) / float(den))


def encode(ctx: CkksContext, slots, scale: Fraction, level: int, p_extend: bool = False) -> Plaintext:
    """encode (ckks.cpp:278-319) on the GPU: slot scatter, the reference's
    radix-2 IDFT, psi^-k twist, rounding and RNS reduction, forward NTT."""
    z = torch.as_tensor(np.asarray(slots, dtype=np.complex128) if not torch.is_tensor(slots) else slots)
    if z.numel() > ctx.n // 2:
        raise ValueError("too many slots")
    if level < 1 or level > ctx.params.l:
        raise ValueError("level out of range")
    if scale <= 0 or log2_rational(Fraction(scale)) > 60.0:
        raise ValueError("scale out of the representable range")
    zr = torch.view_as_real(z.to(torch.complex128).reshape(-1)).contiguous().to(ctx.device)
    rows = level + (ctx.params.alpha if p_extend else 0)
    out = ctx.empty(rows, ctx.n)
    nat.call("ck_encode", ctx.handle, ctypes.c_void_p(zr.data_ptr() if zr.numel() else 0), z.numel(),
             ctypes.c_double(log2_rational(Fraction(scale))), level, int(p_extend), _ptr(out), ctx.stream())
    return Plaintext(Polynomial(out, level, ctx.params.alpha if p_extend else 0), Fraction(scale), level)


def _limbs32(x: int) -> list:
    """little-endian 32-bit words of a non-negative integer (at least one)"""
    out = []
    while True:
        out.append(x & 0xFFFFFFFF)
        x >>= 32
        if not x:
            return out


def decode(ctx: CkksContext, pt: Plaintext) -> np.ndarray:
    """decode (ckks.cpp:321-362) on the GPU -> n/2 complex slots (numpy)."""
    _check_eval_mont(pt.poly, "decode")
    out = torch.empty(ctx.n, dtype=torch.float64, device=ctx.device)
    sc = Fraction(pt.scale)
    num, den = _limbs32(sc.numerator), _limbs32(sc.denominator)
    if len(num) <= 8 and len(den) <= 8:  # the exact rational: slots bit-identical to the reference's
        nat.call("ck_decode_rational", ctx.handle, _ptr(pt.poly.data), pt.level,
                 ctypes.c_double(log2_rational(pt.scale)), nat.u32_array(num), len(num), nat.u32_array(den), len(den),
                 _ptr(out), ctx.stream())
    else:
        nat.call("ck_decode", ctx.handle, _ptr(pt.poly.data), pt.level, ctypes.c_double(log2_rational(pt.scale)),
                 _ptr(out), ctx.stream())
    h = out.cpu().numpy()
    return h[0::2] + 1j * h[1::2]


# ------------------------------------------------------ encrypt / decrypt --
def decrypt(ctx: CkksContext, ct: Ciphertext, s: torch.Tensor) -> Plaintext:
    """decrypt (ckks.cpp:541-553): m = b + a s (evaluation, Montgomery).
    `s` holds at least ct.level rows of the secret (sk.s of the reference)."""
    _check_pair(ctx, ct)
    rows = s[: ct.level].contiguous()
    shape = list(ct.data.shape)
    del shape[-3]
    out = torch.empty(shape, dtype=torch.int32, device=ctx.device)
    nat.call("ck_decrypt", ctx.handle, ct.level, ct.batch, _ptr(ct.data), _ptr(rows), _ptr(out), ctx.stream())
    return Plaintext(Polynomial(out, ct.level, 0), ct.scale, ct.level)


def coeffs_to_eval(ctx: CkksContext, coeffs, level: int, p_rows: int = 0) -> Polynomial:
    """coeffs_to_eval (ckks.cpp:366-380): signed integer coefficients ->
    evaluation-domain Montgomery rows over Q_level (+ p_rows P primes)."""
    c = torch.as_tensor(np.asarray(coeffs, dtype=np.int64) if not torch.is_tensor(coeffs) else coeffs)
    c = c.to(device=ctx.device, dtype=torch.int64).contiguous()
    if c.numel() != ctx.n:
        raise ValueError("need n coefficients")
    out = ctx.empty(level + p_rows, ctx.n)
    nat.call("ck_coeffs_to_eval", ctx.handle, _ptr(c), level, p_rows, _ptr(out), ctx.stream())
    return Polynomial(out, level, p_rows)


def encrypt_sk(ctx: CkksContext, pt: Plaintext, s: torch.Tensor, a: torch.Tensor, e: Polynomial) -> Ciphertext:
    """Secret-key encrypt (ckks.cpp:497-516) with caller-supplied randomness:
    `a` uniform evaluation-domain rows, `e` the Gaussian error in evaluation
    form (coeffs_to_eval).  (b, a) = (m + e - a s, a)."""
    _check_eval_mont(pt.poly, "encrypt")
    if pt.poly.p_count != 0:
        raise ValueError("cannot encrypt a P-extended plaintext")
    l = pt.level
    out = ctx.empty(2, l, ctx.n)
    nat.call("ck_encrypt_sk", ctx.handle, l, _ptr(pt.poly.data[:l].contiguous()), _ptr(a[:l].contiguous()),
             _ptr(e.data[:l].contiguous()), _ptr(s[:l].contiguous()), _ptr(out), ctx.stream())
    return Ciphertext(out, pt.scale, l)


def encrypt_pk(ctx: CkksContext, pt: Plaintext, pk: Ciphertext, v: Polynomial, e0: Polynomial,
               e1: Polynomial) -> Ciphertext:
    """Public-key encrypt (ckks.cpp:518-539) with caller-supplied randomness
    (v ternary, e0 / e1 Gaussian, all in evaluation form):
    (b, a) = (v pk.b + e0 + m, v pk.a + e1)."""
    _check_eval_mont(pt.poly, "encrypt")
    if pt.poly.p_count != 0:
        raise ValueError("cannot encrypt a P-extended plaintext")
    l = pt.level
    pkl = torch.stack([pk.data[0, :l], pk.data[1, :l]]).contiguous()
    out = ctx.empty(2, l, ctx.n)
    nat.call("ck_encrypt_pk", ctx.handle, l, _ptr(pt.poly.data[:l].contiguous()), _ptr(v.data[:l].contiguous()),
             _ptr(e0.data[:l].contiguous()), _ptr(e1.data[:l].contiguous()), _ptr(pkl), _ptr(out), ctx.stream())
    return Ciphertext(out, pt.scale, l)


class RefRng:
    """The reference's randomness: ``std::mt19937_64(seed)`` consumed draw for
    draw as ckks.cpp does (host side, sequential, like the reference; C ABI
    ``ck_rng_*`` / ``ck_sample_*``).  Pass it wherever an ``rng`` is taken and
    keys / ciphertexts come out bit-identical to the reference's for the same
    seed (tests/test_gpu_keys.py against the golden fixtures).  A numpy
    Generator is accepted too (different stream, same distributions)."""

    def __init__(self, seed: int):
        h = ctypes.c_void_p()
        nat.call("ck_rng_create", ctypes.c_uint64(seed), ctypes.byref(h))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            nat.call("ck_rng_destroy", self._h)
            self._h = None

    def draws(self, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        nat.call("ck_rng_draws", self._h, ctypes.c_uint64(count), out.ctypes.data)
        return out

    def gaussian(self, n: int, sigma: float) -> np.ndarray:
        out = np.empty(n, np.int64)
        nat.call("ck_sample_gaussian", self._h, n, ctypes.c_double(sigma), out.ctypes.data)
        return out

    def ternary(self, n: int, h: int) -> np.ndarray:
        out = np.empty(n, np.int64)
        nat.call("ck_sample_ternary", self._h, n, h, out.ctypes.data)
        return out

    def uniform(self, primes: Sequence[int], n: int) -> np.ndarray:
        q = np.ascontiguousarray(np.asarray(primes, np.uint32))
        out = np.empty((len(q), n), np.uint32)
        nat.call("ck_sample_uniform", self._h, q.ctypes.data, len(q), n, out.ctypes.data)
        return out


def keygen(ctx: CkksContext, rng) -> torch.Tensor:
    """keygen (ckks.cpp:399-405): ternary secret of Hamming weight
    params.hamming (host sampling) -> evaluation rows over the full L + alpha
    basis (the reference's sk.s)."""
    c = sample_ternary(ctx.n, min(ctx.params.hamming, ctx.n // 4), rng)
    return coeffs_to_eval(ctx, c, ctx.params.l, ctx.params.alpha).data


def pubkey_gen(ctx: CkksContext, s: torch.Tensor, rng) -> Ciphertext:
    """pubkey_gen (ckks.cpp:407-424): (b, a) = (e - a s, a) at level L."""
    l = ctx.params.l
    zero = Plaintext(Polynomial(torch.zeros((l, ctx.n), dtype=torch.int32, device=ctx.device), l), Fraction(1), l)
    a = uniform_eval(ctx, l, rng)
    return encrypt_sk(ctx, zero, s, a, coeffs_to_eval(ctx, sample_gaussian(ctx.n, ctx.params.sigma, rng), l))


def encrypt(ctx: CkksContext, pt: Plaintext, key, rng) -> Ciphertext:
    """encrypt (ckks.hpp:164-167): `key` is the secret (sk.s rows, a tensor)
    or a public key (Ciphertext); the randomness is drawn in the reference's
    order (secret key: a, then e, ckks.cpp:504-505; public key: v, e0, e1,
    ckks.cpp:523-526) and the arithmetic runs on the GPU."""
    l, n = pt.level, ctx.n
    if isinstance(key, Ciphertext):
        v = coeffs_to_eval(ctx, sample_ternary(n, min(ctx.params.hamming, n // 4), rng), l)
        e0 = coeffs_to_eval(ctx, sample_gaussian(n, ctx.params.sigma, rng), l)
        e1 = coeffs_to_eval(ctx, sample_gaussian(n, ctx.params.sigma, rng), l)
        return encrypt_pk(ctx, pt, key, v, e0, e1)
    _check_eval_mont(pt.poly, "encrypt")
    if pt.poly.p_count != 0:
        raise ValueError("cannot encrypt a P-extended plaintext")
    a = uniform_eval(ctx, l, rng)
    e = coeffs_to_eval(ctx, sample_gaussian(n, ctx.params.sigma, rng), l)
    return encrypt_sk(ctx, pt, key, a, e)


def evk_gen(ctx: CkksContext, s: torch.Tensor, kind: str, rotation: int, rng: np.random.Generator) -> EvaluationKey:
    """evk_gen (ckks.cpp:426-477): digit k encrypts g_k s_src under s_dst over
    PQ, g_k = P * dhat_k * (dhat_k^-1 mod d_k); relinearisation: s_src = s^2,
    s_dst = s; rotation r: s_src = s, s_dst = phi_{-r}(s)."""
    L, A, n = ctx.params.l, ctx.params.alpha, ctx.n
    rows = L + A
    primes = [int(v) for v in ctx.primes[:rows]]
    full = Polynomial(s[:rows].contiguous(), L, A)
    if kind == RELIN:
        s_src, s_dst, square = full.data, full.data, 1
    else:
        s_src, square = full.data, 0
        s_dst = apply_automorphism(ctx, full, -rotation).data
    q_full = 1
    for q in primes[:L]:
        q_full *= q
    P = 1
    for q in primes[L:]:
        P *= q
    D = ctx.num_digits(L)
    out = ctx.empty(D, 2, rows, n)
    for k in range(D):
        dk = 1
        for q in primes[k * A: min((k + 1) * A, L)]:
            dk *= q
        dhat = q_full // dk
        g = P * dhat * pow(dhat, -1, dk)
        gm = [((g % q) << 32) % q for q in primes]
        a_k = _uniform_rows(ctx, primes, rng)  # Q rows then P rows, as uniform_eval(l, alpha)
        e_k = coeffs_to_eval(ctx, sample_gaussian(n, ctx.params.sigma, rng), L, A).data
        out[k, 1] = a_k
        nat.call("ck_evk_digit", ctx.handle, _ptr(s_src), _ptr(s_dst), _ptr(out[k, 1]), _ptr(e_k),
                 nat.u32_array(gm), square, _ptr(out[k, 0]), ctx.stream())
    return EvaluationKey(out, kind, rotation if kind == ROTATION else 0)


# Host-side samplers for the encryption randomness: with a RefRng the
# reference's own stream (bit-exact keys / ciphertexts); with a numpy
# Generator the same distributions from a different stream.
def sample_ternary(n: int, hamming: int, rng) -> np.ndarray:
    if isinstance(rng, RefRng):
        return rng.ternary(n, hamming)
    c = np.zeros(n, np.int64)
    idx = rng.choice(n, size=hamming, replace=False)
    c[idx] = rng.choice(np.array([-1, 1], np.int64), size=hamming)
    return c


def sample_gaussian(n: int, sigma: float, rng) -> np.ndarray:
    if isinstance(rng, RefRng):
        return rng.gaussian(n, sigma)
    return np.rint(rng.normal(0.0, sigma, n)).astype(np.int64)


def _uniform_rows(ctx: CkksContext, primes: Sequence[int], rng) -> torch.Tensor:
    if isinstance(rng, RefRng):
        u = rng.uniform(primes, ctx.n)
    else:
        q = np.asarray(primes, np.int64)[:, None]
        u = rng.integers(0, 1 << 62, (len(primes), ctx.n), dtype=np.int64) % q
    return torch.from_numpy(u.astype(np.int64).astype(np.int32)).to(ctx.device)


def uniform_eval(ctx: CkksContext, level: int, rng) -> torch.Tensor:
    return _uniform_rows(ctx, [int(v) for v in ctx.q_primes[:level]], rng)


# ----------------------------------------------------------- kernel level --
def ntt_forward(ctx: CkksContext, p: Polynomial) -> Polynomial:  # ntt.cpp:288-299
    if p.domain != COEFFICIENT:
        raise ValueError("ntt_forward expects coefficient domain")
    if p.mont:
        raise ValueError("ntt_forward expects plain form (entry merge)")
    g = nat.u32_array(ctx.gidx(p.q_count, p.p_count))
    nat.call("ck_ntt_forward", ctx.handle, _ptr(p.data), p.rows, g, ctx.stream())
    p.domain, p.mont = EVALUATION, True
    return p


def intt_inverse(ctx: CkksContext, p: Polynomial, epilogue_mont: Optional[Sequence[int]] = None) -> Polynomial:
    """ntt.cpp:301-312 (+ the fused part-1 epilogue of NttPlan::inverse_row)."""
    if p.domain != EVALUATION:
        raise ValueError("intt_inverse expects evaluation domain")
    if not p.mont:
        raise ValueError("intt_inverse expects Montgomery form")
    g = nat.u32_array(ctx.gidx(p.q_count, p.p_count))
    e = nat.u32_array(epilogue_mont) if epilogue_mont is not None else None
    nat.call("ck_intt_inverse", ctx.handle, _ptr(p.data), p.rows, g, e, ctx.stream())
    p.domain, p.mont = COEFFICIENT, False
    return p


def bconv(ctx: CkksContext, src: torch.Tensor, src_gidx: Sequence[int], dst_gidx: Sequence[int]) -> torch.Tensor:
    """make_bconv_table + bconv_part2 (bconv.cpp:13-46, 96-174)."""
    out = ctx.empty(len(dst_gidx), ctx.n)
    nat.call("ck_bconv", ctx.handle, _ptr(src), len(src_gidx), nat.u32_array(src_gidx), _ptr(out), len(dst_gidx),
             nat.u32_array(dst_gidx), ctx.stream())
    return out


def mod_switch(ctx: CkksContext, a: Polynomial, src_gidx: Sequence[int], dst_q_count: int,
               dst_p_count: int = 0) -> Polynomial:
    """mod_switch (bconv.cpp:176-213): evaluation-domain rows over `src_gidx`
    -> rows over Q_[0, dst_q) + P_[0, dst_p), evaluation domain, Montgomery."""
    _check_eval_mont(a, "mod_switch")
    if a.rows != len(src_gidx):
        raise ValueError("input rows do not match table source")
    out = ctx.empty(dst_q_count + dst_p_count, ctx.n)
    nat.call("ck_mod_switch", ctx.handle, _ptr(a.data.contiguous()), len(src_gidx), nat.u32_array(src_gidx),
             _ptr(out), dst_q_count, dst_p_count, ctx.stream())
    return Polynomial(out, dst_q_count, dst_p_count)


def galois_for_rotation(n: int, r: int) -> int:
    """5^-r mod 2n (automorphism.cpp:11-23)."""
    return pow(5, (-r) % (n // 2), 2 * n)


def apply_automorphism(ctx: CkksContext, p: Polynomial, r: int, galois: Optional[int] = None) -> Polynomial:
    """apply_automorphism (automorphism.cpp:76-100): rotation by r slots
    (AutomorphismMap::rotation) or, when ``galois`` is given, any Galois
    element (conjugation = 2n - 1); evaluation-domain column gather or the
    coefficient-domain signed permutation."""
    out = torch.empty_like(p.data)
    if galois is None and p.domain == EVALUATION:
        nat.call("ck_automorphism", ctx.handle, _ptr(p.data), _ptr(out), p.rows, int(r), ctx.stream())
    else:
        g = galois_for_rotation(ctx.n, r) if galois is None else int(galois)
        nat.call("ck_automorphism_galois", ctx.handle, _ptr(p.data), _ptr(out), p.q_count, p.p_count, g,
                 int(p.domain == COEFFICIENT), ctx.stream())
    return Polynomial(out, p.q_count, p.p_count, p.domain, p.mont)


EW_ADD, EW_SUB, EW_MUL = 0, 1, 2


def ew_add(ctx: CkksContext, a: Polynomial, b: Polynomial) -> Polynomial:  # poly.cpp:146-150
    return _ew(ctx, EW_ADD, a, b, a.mont)


def ew_sub(ctx: CkksContext, a: Polynomial, b: Polynomial) -> Polynomial:  # poly.cpp:152-156
    return _ew(ctx, EW_SUB, a, b, a.mont)


def ew_mul(ctx: CkksContext, a: Polynomial, b: Polynomial) -> Polynomial:  # poly.cpp:158-164
    if not a.mont or not b.mont:
        raise ValueError("ew_mul expects Montgomery-form operands")
    return _ew(ctx, EW_MUL, a, b, True)


def ew_add_inplace(ctx: CkksContext, a: Polynomial, b: Polynomial) -> Polynomial:  # poly.cpp:182-192
    return _ew(ctx, EW_ADD, a, b, a.mont, out=a)


def ew_sub_inplace(ctx: CkksContext, a: Polynomial, b: Polynomial) -> Polynomial:  # poly.cpp:194-205
    return _ew(ctx, EW_SUB, a, b, a.mont, out=a)


def ew_mul_const(ctx: CkksContext, a: Polynomial, consts_mont: Sequence[int]) -> Polynomial:  # poly.cpp:166-180
    if len(consts_mont) != a.rows:
        raise ValueError("constant count mismatch")
    out = torch.empty_like(a.data)
    nat.call("ck_ew_mul_const", ctx.handle, _ptr(a.data), nat.u32_array([int(c) for c in consts_mont]), _ptr(out),
             a.q_count, a.p_count, ctx.stream())
    return Polynomial(out, a.q_count, a.p_count, a.domain, a.mont)


def _ew(ctx, op, a: Polynomial, b: Polynomial, mont_out: bool, out: Optional[Polynomial] = None) -> Polynomial:
    if a.q_count != b.q_count or a.p_count != b.p_count:  # check_binary, poly.cpp:115-119
        raise ValueError("basis prefix mismatch")
    if a.domain != b.domain:
        raise ValueError("domain mismatch")
    if a.mont != b.mont:
        raise ValueError("Montgomery flag mismatch")
    if out is not None:
        nat.call("ck_ew_binary", ctx.handle, op, _ptr(a.data), _ptr(b.data), _ptr(out.data), a.q_count, a.p_count,
                 ctx.stream())
        return out
    o = torch.empty_like(a.data)
    nat.call("ck_ew_binary", ctx.handle, op, _ptr(a.data), _ptr(b.data), _ptr(o), a.q_count, a.p_count, ctx.stream())
    return Polynomial(o, a.q_count, a.p_count, a.domain, mont_out)


# ------------------------------------------------------------ wire formats --
# Byte-compatible with the reference's serialisers (ckks.cpp:1090-1154,
# poly.cpp:295-352, rns.cpp:168-216) through the C ABI: rows go straight
# between device memory and the blob.
def _blob(fn, args, stream=None) -> bytes:
    """Call a ck_serialize_* writer twice: length query (out = NULL), then fill."""
    tail = [] if stream is None else [stream]
    n = ctypes.c_size_t()
    nat.call(fn, *args, None, 0, ctypes.byref(n), *tail)
    buf = ctypes.create_string_buffer(max(1, n.value))
    nat.call(fn, *args, buf, n.value, ctypes.byref(n), *tail)
    return buf.raw[: n.value]


def _be(v: int) -> bytes:
    return v.to_bytes(max(1, (v.bit_length() + 7) // 8), "big")


def serialize_basis(ctx: CkksContext) -> bytes:  # rns.cpp:188-199
    return _blob("ck_serialize_basis", [ctx.handle])


def serialize_poly(ctx: CkksContext, p: Polynomial) -> bytes:  # poly.cpp:297-320
    return _blob("ck_serialize_poly", [ctx.handle, _ptr(p.data.contiguous()), p.q_count, p.p_count,
                                       int(p.domain == EVALUATION), int(p.mont)], ctx.stream())


def deserialize_poly(ctx: CkksContext, blob: bytes) -> Polynomial:  # poly.cpp:322-352
    out = ctx.empty(ctx.params.l + ctx.params.alpha, ctx.n)
    meta = (ctypes.c_uint32 * 4)()
    nat.call("ck_deserialize_poly", ctx.handle, blob, len(blob), _ptr(out), out.shape[0], meta, ctx.stream())
    qc, pc, dom, mont = list(meta)
    return Polynomial(out[: qc + pc].clone(), qc, pc, EVALUATION if dom else COEFFICIENT, bool(mont))


def serialize_ciphertext(ctx: CkksContext, ct: Ciphertext) -> bytes:  # ckks.cpp:1092-1105
    if ct.batched:
        raise ValueError("serialize one ciphertext at a time")
    s = Fraction(ct.scale)
    num, den = _be(s.numerator), _be(s.denominator)
    return _blob("ck_serialize_ciphertext", [ctx.handle, _ptr(ct.data.contiguous()), ct.level,
                                             int(ct.pending_rescale), num, len(num), den, len(den)], ctx.stream())


def deserialize_ciphertext(ctx: CkksContext, blob: bytes) -> Ciphertext:  # ckks.cpp:1107-1121
    out = ctx.empty(2, ctx.params.l, ctx.n)
    lv, pend = ctypes.c_uint32(), ctypes.c_int()
    nb, db = ctypes.create_string_buffer(len(blob)), ctypes.create_string_buffer(len(blob))
    nl, dl = ctypes.c_size_t(), ctypes.c_size_t()
    flat = out.view(-1)
    nat.call("ck_deserialize_ciphertext", ctx.handle, blob, len(blob), _ptr(flat), ctx.params.l, ctypes.byref(lv),
             ctypes.byref(pend), nb, len(blob), ctypes.byref(nl), db, len(blob), ctypes.byref(dl), ctx.stream())
    level = lv.value
    data = flat[: 2 * level * ctx.n].view(2, level, ctx.n).clone()
    scale = Fraction(int.from_bytes(nb.raw[: nl.value], "big"), int.from_bytes(db.raw[: dl.value], "big"))
    return Ciphertext(data, scale, level, bool(pend.value))


def serialize_evk(ctx: CkksContext, evk: "EvaluationKey") -> bytes:  # ckks.cpp:1123-1137
    D = evk.data.shape[0]
    return _blob("ck_serialize_evk", [ctx.handle, _ptr(evk.data.contiguous()), D, 0 if evk.kind == RELIN else 1,
                                      int(evk.rotation)], ctx.stream())


def deserialize_evk(ctx: CkksContext, blob: bytes) -> "EvaluationKey":  # ckks.cpp:1139-1154
    D = ctx.num_digits(ctx.params.l)
    out = ctx.empty(D, 2, ctx.params.l + ctx.params.alpha, ctx.n)
    kind, rot, d = ctypes.c_int(), ctypes.c_int64(), ctypes.c_uint32()
    nat.call("ck_deserialize_evk", ctx.handle, blob, len(blob), _ptr(out), D, ctypes.byref(kind), ctypes.byref(rot),
             ctypes.byref(d), ctx.stream())
    return EvaluationKey(out[: d.value].contiguous(), RELIN if kind.value == 0 else ROTATION, rot.value)
