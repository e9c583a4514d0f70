"""Helpers shared by the CPU and GPU parity tests: golden fixture loading."""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

from paper_2407_13055_b200 import wire

GOLDEN = Path(__file__).resolve().parent / "golden"
SMALL_DIRS = sorted(p for p in GOLDEN.glob("small_*") if p.is_dir())
FULL = json.loads((GOLDEN / "full_hashes.json").read_text())


# fixture seeds of tests/golden/make_golden.py SMALL: (n, l, alpha) -> seed
SMALL_SEEDS = {(256, 6, 2): 42, (1024, 8, 3): 43, (512, 4, 8): 44}


def ref_unit_slots(draws: np.ndarray) -> np.ndarray:
    """std::uniform_real_distribution<double>(-1, 1) over mt19937_64 draws
    as libstdc++ evaluates it (generate_canonical<double, 53>: one draw,
    double(x) / 2^64, clamped below 1; then (b - a) * r + a), two draws per
    complex slot (re, im) -- oracle/ref_driver.cpp unit_slots."""
    r = np.array([float(int(x)) for x in draws]) / 18446744073709551616.0  # correctly rounded
    r = np.where(r >= 1.0, np.nextafter(1.0, 0.0), r)
    v = 2.0 * r + (-1.0)
    return v[0::2] + 1j * v[1::2]


def parse_small_name(d: Path):
    _, n, l, a = d.name.split("_")
    return int(n[1:]), int(l[1:]), int(a[1:])


class Fixture:
    def __init__(self, d: Path):
        self.dir = d
        self.basis = wire.read_basis((d / "basis.bin").read_bytes())
        self.n, self.l, self.alpha, self.db = self.basis.n, self.basis.l, self.basis.alpha, self.basis.delta_bits

    def ct(self, name):
        return wire.read_ciphertext((self.dir / f"{name}.bin").read_bytes())

    def poly(self, name):
        return wire.read_poly((self.dir / f"{name}.bin").read_bytes())[0]

    def evk(self, name):
        return wire.read_evk((self.dir / f"{name}.bin").read_bytes())

    @staticmethod
    def ct_rows(ct):
        return np.stack([ct.b.rows, ct.a.rows])


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u4").tobytes()).hexdigest()


def full_cases():
    cases = []
    for name, cfg in FULL["configs"].items():
        for key, h in cfg["ops"].items():
            op, level, rot = key.split("@")
            cases.append((name, cfg, op, int(level), int(rot), h))
    return cases
