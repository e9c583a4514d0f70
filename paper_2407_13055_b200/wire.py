"""Byte-compatible readers/writers for the reference's versioned wire formats
(SURVEY.md §8f item 2), so ciphertexts, keys, polynomials and bases move
between the CPU reference and the GPU without conversion:

  basis       "RBS1"  rns.cpp:168-216
  polynomial  "PLS1"  poly.cpp:295-352 (rows are canonical little-endian u32)
  ciphertext  "CTS1"  ckks.cpp:1090-1121 (rational scale as big-int bytes)
  eval key    "EVK1"  ckks.cpp:1123-1154
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from fractions import Fraction
from typing import List, Tuple

import numpy as np

POLY_MAGIC, BASIS_MAGIC, CT_MAGIC, EVK_MAGIC = 0x31534C50, 0x31534252, 0x31535443, 0x314B5645


def basis_hash(n: int, delta_bits: int, q_primes, p_primes) -> int:
    """RnsBasis::hash (rns.cpp:119-133): FNV-1a over little-endian u64 words."""
    h = 1469598103934665603
    mask = (1 << 64) - 1

    def mix(v):
        nonlocal h
        for i in range(8):
            h ^= (v >> (8 * i)) & 0xFF
            h = (h * 1099511628211) & mask

    mix(n)
    mix(delta_bits)
    for q in q_primes:
        mix(int(q))
    mix(mask)
    for p in p_primes:
        mix(int(p))
    return h


@dataclass
class PolyBlob:
    n: int
    q_count: int
    p_count: int
    domain: int  # 0 coefficient, 1 evaluation
    mont: bool
    basis_hash: int
    rows: np.ndarray  # [q_count + p_count, n] uint32 canonical


def read_poly(b: bytes, off: int = 0) -> Tuple[PolyBlob, int]:
    magic, n, qc, pc, dom, mont, hlo, hhi = struct.unpack_from("<8I", b, off)
    if magic != POLY_MAGIC:
        raise RuntimeError("bad polynomial magic")
    off += 32
    cnt = (qc + pc) * n
    if off + 4 * cnt > len(b):
        raise RuntimeError("truncated polynomial blob")
    rows = np.frombuffer(b, dtype="<u4", count=cnt, offset=off).reshape(qc + pc, n).copy()
    return PolyBlob(n, qc, pc, dom, bool(mont), hlo | (hhi << 32), rows), off + 4 * cnt


def write_poly(p: PolyBlob) -> bytes:
    h = p.basis_hash
    head = struct.pack("<8I", POLY_MAGIC, p.n, p.q_count, p.p_count, p.domain, int(p.mont), h & 0xFFFFFFFF, h >> 32)
    return head + np.ascontiguousarray(p.rows, dtype="<u4").tobytes()


def _read_bigint(b: bytes, off: int) -> Tuple[int, int]:
    (ln,) = struct.unpack_from("<I", b, off)
    off += 4
    if off + 1 + ln > len(b):
        raise ValueError("truncated input")
    neg = b[off] != 0
    off += 1
    v = int.from_bytes(b[off:off + ln], "big") if ln else 0
    return (-v if neg else v), off + ln


def _write_bigint(v: int) -> bytes:
    mag = abs(v)
    by = mag.to_bytes(max(1, (mag.bit_length() + 7) // 8), "big")  # export_bits msv-first; 0 -> one 0 byte
    return struct.pack("<I", len(by)) + bytes([1 if v < 0 else 0]) + by


def _read_sized_poly(b: bytes, off: int) -> Tuple[PolyBlob, int]:
    (ln,) = struct.unpack_from("<Q", b, off)
    off += 8
    if off + ln > len(b):
        raise ValueError("truncated input")
    p, _ = read_poly(b[off:off + ln])
    return p, off + ln


def _write_sized_poly(p: PolyBlob) -> bytes:
    blob = write_poly(p)
    return struct.pack("<Q", len(blob)) + blob


@dataclass
class CiphertextBlob:
    level: int
    pending_rescale: bool
    scale: Fraction
    b: PolyBlob
    a: PolyBlob


def read_ciphertext(b: bytes) -> CiphertextBlob:
    magic, ver, level = struct.unpack_from("<3I", b, 0)
    if magic != CT_MAGIC or ver != 1:
        raise ValueError("bad ciphertext header")
    off = 12
    pending = b[off] != 0
    off += 1
    num, off = _read_bigint(b, off)
    den, off = _read_bigint(b, off)
    if den == 0:
        raise ValueError("zero denominator")
    pb, off = _read_sized_poly(b, off)
    pa, off = _read_sized_poly(b, off)
    return CiphertextBlob(level, pending, Fraction(num, den), pb, pa)


def write_ciphertext(ct: CiphertextBlob) -> bytes:
    s = Fraction(ct.scale)
    out = struct.pack("<3I", CT_MAGIC, 1, ct.level) + bytes([1 if ct.pending_rescale else 0])
    out += _write_bigint(s.numerator) + _write_bigint(s.denominator)
    return out + _write_sized_poly(ct.b) + _write_sized_poly(ct.a)


@dataclass
class EvkBlob:
    kind: int  # 0 relin, 1 rotation
    rotation: int
    digits: List[Tuple[PolyBlob, PolyBlob]]

    def stacked(self) -> np.ndarray:
        """[D, 2, L+alpha, n] uint32 — the layout of include/ck32_b200.h."""
        return np.stack([np.stack([b.rows, a.rows]) for b, a in self.digits])


def read_evk(b: bytes) -> EvkBlob:
    magic, ver, kind = struct.unpack_from("<3I", b, 0)
    if magic != EVK_MAGIC or ver != 1:
        raise ValueError("bad key header")
    (rot,) = struct.unpack_from("<q", b, 12)
    (d,) = struct.unpack_from("<I", b, 20)
    off = 24
    digits = []
    for _ in range(d):
        pb, off = _read_sized_poly(b, off)
        pa, off = _read_sized_poly(b, off)
        digits.append((pb, pa))
    return EvkBlob(kind, rot, digits)


def write_evk(e: EvkBlob) -> bytes:
    out = struct.pack("<3IqI", EVK_MAGIC, 1, e.kind, e.rotation, len(e.digits))
    for pb, pa in e.digits:
        out += _write_sized_poly(pb) + _write_sized_poly(pa)
    return out


@dataclass
class BasisBlob:
    n: int
    l: int
    alpha: int
    delta_bits: int
    primes: np.ndarray  # Q then P

    @property
    def hash(self) -> int:
        return basis_hash(self.n, self.delta_bits, self.primes[: self.l], self.primes[self.l:])


def read_basis(b: bytes) -> BasisBlob:
    if len(b) < 24:
        raise RuntimeError("truncated basis blob")
    magic, ver, n, l, alpha, db = struct.unpack_from("<6I", b, 0)
    if magic != BASIS_MAGIC:
        raise RuntimeError("bad basis magic")
    if ver != 1:
        raise RuntimeError("bad basis version")
    if len(b) < 24 + 4 * (l + alpha):
        raise RuntimeError("truncated basis blob")
    primes = np.frombuffer(b, dtype="<u4", count=l + alpha, offset=24).copy()
    return BasisBlob(n, l, alpha, db, primes)


def write_basis(bb: BasisBlob) -> bytes:
    return struct.pack("<6I", BASIS_MAGIC, 1, bb.n, bb.l, bb.alpha, bb.delta_bits) + \
        np.ascontiguousarray(bb.primes, "<u4").tobytes()
