"""ORACLE TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

* :class:`Oracle` wraps ``oracle/_ref/libck32_oracle.so``, the in-repo C
  restatement of the reference hot path (``oracle/ck32_oracle.c``).  It is
  built from repo sources only, so it exists on the GPU box too.
* :class:`Reference` wraps ``oracle/_ref/libckks32_ref_driver.so``: the
  reference itself (``/root/reference/proj/src``) compiled read-only with the
  Boost shim (``oracle/Makefile``).  Present wherever ``oracle/_ref`` was built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
ORACLE_SO = REF_DIR / "libck32_oracle.so"
REF_SO = REF_DIR / "libckks32_ref_driver.so"
REF_SO_NDEBUG = REF_DIR / "libckks32_ref_nd_driver.so"

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_vp = ctypes.c_void_p


def build_oracle() -> Path:
    """Compile the C restatement (repo sources only) if it is missing."""
    if not ORACLE_SO.exists():
        subprocess.run(["make", "-C", str(HERE), "restate"], check=True, capture_output=True)
    return ORACLE_SO


_olib = None


def _oracle_lib():
    global _olib
    if _olib is None:
        lib = ctypes.CDLL(str(build_oracle()))
        lib.cko_create.restype = _vp
        lib.cko_create.argtypes = [ctypes.c_uint32] * 4
        lib.cko_destroy.argtypes = [_vp]
        lib.cko_primes.restype = ctypes.POINTER(ctypes.c_uint32)
        lib.cko_primes.argtypes = [_vp]
        lib.cko_generate_basis.argtypes = [ctypes.c_uint32] * 4 + [_u32p]
        lib.cko_twiddles.argtypes = [_vp, ctypes.c_uint32, _u32p, _u32p, _u32p]
        lib.cko_rng_seed.argtypes = [_vp, ctypes.c_uint64]
        lib.cko_rng_next.restype = ctypes.c_uint64
        lib.cko_rng_next.argtypes = [_vp]
        lib.cko_random_rows.argtypes = [_vp, _vp, ctypes.c_uint32, _u32p, _i32p]
        lib.cko_ntt_fwd_row.argtypes = [_vp, _i32p, ctypes.c_uint32]
        lib.cko_intt_row.argtypes = [_vp, _i32p, ctypes.c_uint32, _vp]
        lib.cko_bconv.argtypes = [_vp, ctypes.c_uint32, _u32p, ctypes.c_uint32, _u32p, _i32p, _i32p]
        lib.cko_bconv_part1.argtypes = [_vp, ctypes.c_uint32, _u32p, _u32p]
        lib.cko_mod_up.argtypes = [_vp, ctypes.c_uint32, _i32p, _i32p]
        lib.cko_key_mult.argtypes = [_vp, ctypes.c_uint32, _i32p, _i32p, _i32p, _i32p]
        lib.cko_mod_down.argtypes = [_vp, ctypes.c_uint32, _i32p, _i32p]
        lib.cko_key_switch.argtypes = [_vp, ctypes.c_uint32, _i32p, _i32p, _i32p, _i32p]
        lib.cko_rescale.argtypes = [_vp, ctypes.c_uint32, _i32p, _i32p, _i32p, _i32p]
        lib.cko_hmult.argtypes = [_vp, ctypes.c_uint32, _i32p, _i32p, _i32p, _i32p, _i32p, ctypes.c_int, _i32p, _i32p]
        lib.cko_hrot.argtypes = [_vp, ctypes.c_uint32, _i32p, _i32p, ctypes.c_int64, _i32p, _i32p, _i32p]
        lib.cko_rotation_src_map.argtypes = [ctypes.c_uint32, ctypes.c_int64, _u32p]
        lib.cko_ew_add.argtypes = [_vp, ctypes.c_uint32, _i32p, _i32p, _i32p]
        lib.cko_ew_mul.argtypes = [_vp, ctypes.c_uint32, _i32p, _i32p, _i32p]
        lib.cko_ew_rows.argtypes = [_vp, ctypes.c_int, ctypes.c_uint32, _u32p, _i32p, _i32p, _vp, _i32p]
        lib.cko_automorphism.argtypes = [_vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, _i32p,
                                         _i32p]
        lib.cko_hoisted_accumulate.argtypes = [_vp, ctypes.c_uint32, _i32p, _i32p, ctypes.c_uint32,
                                               ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_vp),
                                               ctypes.POINTER(_vp), _i32p, _i32p]
        _olib = lib
    return _olib


class Rng:
    """std::mt19937_64 (the reference's generator, bench.cpp:121-129)."""

    def __init__(self, seed: int):
        self._lib = _oracle_lib()
        self._state = ctypes.create_string_buffer(312 * 8 + 16)
        self._lib.cko_rng_seed(self._state, seed)

    def next(self) -> int:
        return self._lib.cko_rng_next(self._state)


def generate_basis(n: int, l: int, alpha: int, delta_bits: int) -> np.ndarray:
    out = np.zeros(l + alpha, np.uint32)
    if _oracle_lib().cko_generate_basis(n, l, alpha, delta_bits, out) != 0:
        raise ValueError("basis exhausted")
    return out


class Oracle:
    """C restatement of the reference hot path (see oracle/ck32_oracle.h)."""

    def __init__(self, n: int, l: int, alpha: int, delta_bits: int = 55):
        self.lib = _oracle_lib()
        self.n, self.l, self.alpha, self.delta_bits = n, l, alpha, delta_bits
        self._c = self.lib.cko_create(n, l, alpha, delta_bits)
        if not self._c:
            raise ValueError("basis exhausted")
        p = self.lib.cko_primes(self._c)
        self.primes = np.array([p[i] for i in range(l + alpha)], dtype=np.uint32)

    def __del__(self):
        if getattr(self, "_c", None):
            self.lib.cko_destroy(self._c)
            self._c = None

    # -- helpers --------------------------------------------------------
    def digits(self, level: int) -> int:
        return (level + self.alpha - 1) // self.alpha

    def gidx(self, level: int, p_rows: int = 0) -> np.ndarray:
        return np.concatenate([np.arange(level), self.l + np.arange(p_rows)]).astype(np.uint32)

    def canonical(self, a: np.ndarray, gidx: np.ndarray) -> np.ndarray:
        q = self.primes[gidx].astype(np.int64)[:, None]
        return (a.reshape(len(gidx), -1).astype(np.int64) % q).astype(np.uint32)

    def random_rows(self, rng: Rng, gidx: np.ndarray) -> np.ndarray:
        out = np.zeros((len(gidx), self.n), np.int32)
        self.lib.cko_random_rows(self._c, rng._state, len(gidx), np.ascontiguousarray(gidx, np.uint32), out)
        return out

    def synthetic(self, level: int, seed: int):
        """Inputs of ref_synthetic_op (oracle/ref_driver.cpp): x.b, x.a, y.b,
        y.a (level rows) then the evk [D(L)][2][L+alpha][n]."""
        rng = Rng(seed)
        q = self.gidx(level)
        xb, xa, yb, ya = (self.random_rows(rng, q) for _ in range(4))
        full = self.gidx(self.l, self.alpha)
        D = self.digits(self.l)
        evk = np.zeros((D, 2, self.l + self.alpha, self.n), np.int32)
        for k in range(D):
            evk[k, 0] = self.random_rows(rng, full)
            evk[k, 1] = self.random_rows(rng, full)
        return xb, xa, yb, ya, evk

    def twiddles(self, g: int):
        fwd = np.zeros(self.n, np.uint32)
        inv = np.zeros(self.n, np.uint32)
        s = np.zeros(4, np.uint32)
        self.lib.cko_twiddles(self._c, g, fwd, inv, s)
        return fwd, inv, s

    # -- kernels --------------------------------------------------------
    def ntt_fwd(self, rows: np.ndarray, gidx) -> np.ndarray:
        out = np.ascontiguousarray(rows, np.int32).copy().reshape(len(gidx), self.n)
        for i, g in enumerate(gidx):
            r = np.ascontiguousarray(out[i])
            self.lib.cko_ntt_fwd_row(self._c, r, int(g))
            out[i] = r
        return out

    def intt(self, rows: np.ndarray, gidx, epilogue=None) -> np.ndarray:
        out = np.ascontiguousarray(rows, np.int32).copy().reshape(len(gidx), self.n)
        for i, g in enumerate(gidx):
            r = np.ascontiguousarray(out[i])
            if epilogue is None:
                self.lib.cko_intt_row(self._c, r, int(g), None)
            else:
                e = ctypes.c_uint32(int(epilogue[i]))
                self.lib.cko_intt_row(self._c, r, int(g), ctypes.byref(e))
            out[i] = r
        return out

    def bconv(self, src: np.ndarray, src_gidx, dst_gidx) -> np.ndarray:
        sg = np.ascontiguousarray(src_gidx, np.uint32)
        dg = np.ascontiguousarray(dst_gidx, np.uint32)
        out = np.zeros((len(dg), self.n), np.int32)
        self.lib.cko_bconv(self._c, len(sg), sg, len(dg), dg, np.ascontiguousarray(src, np.int32), out)
        return out

    def bconv_part1(self, src_gidx) -> np.ndarray:
        sg = np.ascontiguousarray(src_gidx, np.uint32)
        out = np.zeros(len(sg), np.uint32)
        self.lib.cko_bconv_part1(self._c, len(sg), sg, out)
        return out

    def mod_up(self, level: int, d: np.ndarray) -> np.ndarray:
        out = np.zeros((self.digits(level), level + self.alpha, self.n), np.int32)
        self.lib.cko_mod_up(self._c, level, np.ascontiguousarray(d, np.int32), out)
        return out

    def key_mult(self, level: int, hoist: np.ndarray, evk: np.ndarray):
        v0 = np.zeros((level + self.alpha, self.n), np.int32)
        v1 = np.zeros_like(v0)
        self.lib.cko_key_mult(self._c, level, np.ascontiguousarray(hoist, np.int32), np.ascontiguousarray(evk, np.int32), v0, v1)
        return v0, v1

    def mod_down(self, level: int, v: np.ndarray) -> np.ndarray:
        out = np.zeros((level, self.n), np.int32)
        self.lib.cko_mod_down(self._c, level, np.ascontiguousarray(v, np.int32), out)
        return out

    def key_switch(self, level: int, d, evk):
        c0 = np.zeros((level, self.n), np.int32)
        c1 = np.zeros_like(c0)
        self.lib.cko_key_switch(self._c, level, np.ascontiguousarray(d, np.int32), np.ascontiguousarray(evk, np.int32), c0, c1)
        return c0, c1

    def rescale(self, level: int, b, a):
        ob = np.zeros((level - 2, self.n), np.int32)
        oa = np.zeros_like(ob)
        if self.lib.cko_rescale(self._c, level, np.ascontiguousarray(b, np.int32), np.ascontiguousarray(a, np.int32), ob, oa):
            raise ValueError("level exhausted")
        return ob, oa

    def hmult(self, level: int, xb, xa, yb, ya, evk, lazy: bool = False):
        lo = level if lazy else level - 2
        ob = np.zeros((lo, self.n), np.int32)
        oa = np.zeros_like(ob)
        c = lambda a: np.ascontiguousarray(a, np.int32)
        if self.lib.cko_hmult(self._c, level, c(xb), c(xa), c(yb), c(ya), c(evk), int(lazy), ob, oa):
            raise ValueError("level exhausted")
        return ob, oa

    def hrot(self, level: int, b, a, r: int, evk):
        ob = np.zeros((level, self.n), np.int32)
        oa = np.zeros_like(ob)
        c = lambda x: np.ascontiguousarray(x, np.int32)
        self.lib.cko_hrot(self._c, level, c(b), c(a), r, c(evk), ob, oa)
        return ob, oa

    def hoisted_accumulate(self, level: int, b, a, rots, pts, evks):
        cnt = len(rots)
        ra = (ctypes.c_int64 * cnt)(*rots)
        keep = [np.ascontiguousarray(p, np.int32) for p in pts]
        ekeep = [np.ascontiguousarray(e, np.int32) if e is not None else None for e in evks]
        pa = (_vp * cnt)(*[k.ctypes.data for k in keep])
        ea = (_vp * cnt)(*[(k.ctypes.data if k is not None else None) for k in ekeep])
        ob = np.zeros((level, self.n), np.int32)
        oa = np.zeros_like(ob)
        c = lambda x: np.ascontiguousarray(x, np.int32)
        self.lib.cko_hoisted_accumulate(self._c, level, c(b), c(a), cnt, ra, pa, ea, ob, oa)
        return ob, oa

    def ew(self, op: int, x: np.ndarray, y, gidx, consts=None) -> np.ndarray:
        """ew_add/sub/mul/mul_const (op 0..3, poly.cpp:121-180) over rows at gidx."""
        g = np.ascontiguousarray(gidx, np.uint32)
        x = np.ascontiguousarray(x, np.int32)
        y = np.ascontiguousarray(x if y is None else y, np.int32)
        k = None if consts is None else np.ascontiguousarray(consts, np.uint32)
        o = np.zeros_like(x)
        self.lib.cko_ew_rows(self._c, op, len(g), g, x, y, None if k is None else k.ctypes.data, o)
        return o

    def automorphism(self, x: np.ndarray, galois: int, coeff: bool) -> np.ndarray:
        """apply_automorphism (automorphism.cpp:76-100) for a Galois element."""
        gi = pow(int(galois), -1, 2 * self.n)
        x = np.ascontiguousarray(x, np.int32)
        o = np.zeros_like(x)
        self.lib.cko_automorphism(self._c, x.shape[0], int(galois), gi, int(coeff), x, o)
        return o

    def rotation_src_map(self, r: int) -> np.ndarray:
        out = np.zeros(self.n, np.uint32)
        self.lib.cko_rotation_src_map(self.n, r, out)
        return out


class Reference:
    """The reference library itself, compiled read-only (oracle/_ref)."""

    available = REF_SO.exists()

    def __init__(self, ndebug: bool = False):
        """ndebug=False: the reference as shipped (-O3, asserts live,
        proj/CMakeLists.txt:10); ndebug=True: the same sources with -DNDEBUG
        (make -C oracle ref-ndebug)."""
        so = REF_SO_NDEBUG if ndebug else REF_SO
        if not so.exists():
            raise FileNotFoundError(f"{so} not built (make -C oracle ref{'-ndebug' if ndebug else ''} "
                                    f"needs /root/reference)")
        lib = ctypes.CDLL(str(so))
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_basis.argtypes = [ctypes.c_uint32] * 4 + [_u32p]
        lib.ref_twiddles.argtypes = [ctypes.c_uint32] * 5 + [_u32p, _u32p, _u32p]
        lib.ref_ntt_rows.argtypes = [ctypes.c_uint32] * 4 + [ctypes.c_int, ctypes.c_uint32, _u32p, _i32p, _vp]
        lib.ref_gen_fixtures.argtypes = [ctypes.c_uint32] * 4 + [ctypes.c_uint64, ctypes.c_char_p]
        lib.ref_synthetic_op.argtypes = [ctypes.c_uint32] * 5 + [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int64,
                                                                  _u32p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
        lib.ref_mechanism_bench.argtypes = [ctypes.c_char_p] + [ctypes.c_uint32] * 7 + [
            ctypes.c_uint64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
            ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_uint64)]
        _f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        lib.ref_encode.argtypes = [ctypes.c_uint32] * 4 + [_f64p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                                           ctypes.c_uint32, ctypes.c_int, _u32p, ctypes.c_size_t]
        lib.ref_decode.argtypes = [ctypes.c_uint32] * 4 + [_u32p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                                           _f64p]
        lib.ref_decode_big.argtypes = [ctypes.c_uint32] * 4 + [_u32p, ctypes.c_uint32, _u32p, ctypes.c_uint32, _u32p,
                                                               ctypes.c_uint32, _f64p]
        self.lib = lib

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def basis(self, n, l, alpha, db=55):
        out = np.zeros(l + alpha, np.uint32)
        self._check(self.lib.ref_basis(n, l, alpha, db, out))
        return out

    def twiddles(self, n, l, alpha, db, g):
        fwd = np.zeros(n, np.uint32)
        inv = np.zeros(n, np.uint32)
        s = np.zeros(4, np.uint32)
        self._check(self.lib.ref_twiddles(n, l, alpha, db, g, fwd, inv, s))
        return fwd, inv, s

    def ntt_rows(self, n, l, alpha, db, rows, gidx, inverse=False, epilogue=None):
        data = np.ascontiguousarray(rows, np.int32).copy()
        g = np.ascontiguousarray(gidx, np.uint32)
        ep = np.ascontiguousarray(epilogue, np.uint32) if epilogue is not None else None
        self._check(self.lib.ref_ntt_rows(n, l, alpha, db, int(inverse), len(g), g, data,
                                          ep.ctypes.data if ep is not None else None))
        return data

    def gen_fixtures(self, n, l, alpha, db, seed, outdir):
        os.makedirs(outdir, exist_ok=True)
        self._check(self.lib.ref_gen_fixtures(n, l, alpha, db, seed, str(outdir).encode()))

    def synthetic_op(self, n, l, alpha, db, level, op, seed, rot=0):
        cap = 4 * (l + alpha) * (l + alpha) * n
        out = np.zeros(cap, np.uint32)
        w = ctypes.c_size_t()
        self._check(self.lib.ref_synthetic_op(n, l, alpha, db, level, op.encode(), seed, rot, out, cap, ctypes.byref(w)))
        return out[: w.value].copy()

    def encode(self, n, l, alpha, db, slots, num, den, level, p_extend=False):
        """reference encode (ckks.cpp:278-319) -> canonical plaintext rows"""
        z = np.asarray(slots, np.complex128)
        flat = np.ascontiguousarray(np.stack([z.real, z.imag], -1).reshape(-1))
        rows = level + (alpha if p_extend else 0)
        out = np.zeros(rows * n, np.uint32)
        self._check(self.lib.ref_encode(n, l, alpha, db, flat, len(z), num, den, level, int(p_extend), out, out.size))
        return out.reshape(rows, n)

    def decode(self, n, l, alpha, db, rows, level, num, den):
        """reference decode (ckks.cpp:321-362) of canonical evaluation-domain rows"""
        out = np.zeros(n, np.float64)
        if num < 1 << 64 and den < 1 << 64:
            self._check(self.lib.ref_decode(n, l, alpha, db, np.ascontiguousarray(rows[:level], np.uint32), level,
                                            num, den, out))
        else:  # multi-word scale (what chains of rescales produce)
            def limbs(x):
                w = []
                while True:
                    w.append(x & 0xFFFFFFFF)
                    x >>= 32
                    if not x:
                        return np.array(w, np.uint32)
            wn, wd = limbs(num), limbs(den)
            self._check(self.lib.ref_decode_big(n, l, alpha, db, np.ascontiguousarray(rows[:level], np.uint32), level,
                                                wn, len(wn), wd, len(wd), out))
        return out[0::2] + 1j * out[1::2]

    def mechanism_bench(self, op, n, l, alpha, db, level, reps, warmup, seed=42):
        med, mn = ctypes.c_double(), ctypes.c_double()
        th = ctypes.c_int()
        cnt = (ctypes.c_uint64 * 7)()
        self._check(self.lib.ref_mechanism_bench(op.encode(), n, l, alpha, db, level, reps, warmup, seed,
                                                 ctypes.byref(med), ctypes.byref(mn), ctypes.byref(th), cnt))
        keys = ["modup", "moddown", "ntt", "intt", "keymult", "bconv", "rescale"]
        return {"median_ns": med.value, "min_ns": mn.value, "omp_threads": th.value,
                "counters": dict(zip(keys, list(cnt)))}
