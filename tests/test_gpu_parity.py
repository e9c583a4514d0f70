"""GPU parity suite: every CUDA result is compared, canonical residue by
residue, with (a) the reference's own fixtures / full-size hashes and (b) the
C restatement oracle on seeded inputs.  Bit-exact is the only bar: all of
this path is integer arithmetic."""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

from golden_util import FULL, SMALL_DIRS, Fixture, full_cases, sha

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2407_13055_b200 import ckks  # noqa: E402
from pyoracle import Oracle, Rng  # noqa: E402

_CTX = {}


def ctx_for(n, l, a, db=55, lazy=False):
    key = (n, l, a, db, lazy)
    if key not in _CTX:
        _CTX[key] = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db, lazy_rescale=lazy))
    return _CTX[key]


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x).astype(np.int32))).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.uint32)


def canon(O, rows, level, p_rows=0):
    return O.canonical(rows, O.gidx(level, p_rows))


def ct(data, level, scale=Fraction(1 << 55)):
    return ckks.Ciphertext(dev(data), scale, level)


# -------------------------------------------------------------- kernel level --
@pytest.mark.parametrize("n", [8, 16, 64, 256, 1024, 4096, 32768, 65536, 131072])
def test_ntt_roundtrip_and_oracle(n):
    l, a = 4, 2
    C = ctx_for(n, l, a, 48)
    O = Oracle(n, l, a, 48)
    rng = Rng(n)
    g = O.gidx(l, a)
    x = O.random_rows(rng, g)
    p = ckks.Polynomial(dev(x), l, a, ckks.COEFFICIENT, False)
    ckks.ntt_forward(C, p)
    np.testing.assert_array_equal(host(p.data), canon(O, O.ntt_fwd(x, g), l, a))
    ckks.intt_inverse(C, p)
    np.testing.assert_array_equal(host(p.data), x.astype(np.uint32))


@pytest.mark.parametrize("n", [256, 65536])
def test_intt_fused_part1_epilogue(n):
    l, a = 6, 3
    C = ctx_for(n, l, a, 48)
    O = Oracle(n, l, a, 48)
    g = O.gidx(l)
    x = O.random_rows(Rng(7), g)
    epi_mont = [int(v) for v in O.bconv_part1(g)]  # part1 constants, Montgomery form (bconv.hpp:22-23)
    p = ckks.Polynomial(dev(x), l, 0)
    ckks.intt_inverse(C, p, epi_mont)
    want = canon(O, O.intt(x, g, epi_mont), l)
    np.testing.assert_array_equal(host(p.data), want)


@pytest.mark.parametrize("n", [1024, 65536])
@pytest.mark.parametrize("shape", [(8, 24), (10, 22), (2, 22), (1, 3), (16, 40)])
def test_bconv_matches_oracle(n, shape):
    sc, dc = shape
    l, a = 40, 16
    if sc == 16:
        a = 16
    C = ctx_for(n, l, a, 48)
    O = Oracle(n, l, a, 48)
    src_g = list(range(l - sc, l)) if sc <= 10 else [l + j for j in range(sc)]
    dst_g = list(range(dc))
    src = O.canonical(O.random_rows(Rng(sc * 100 + dc), np.array(src_g, np.uint32)), np.array(src_g, np.uint32))
    got = ckks.bconv(C, dev(src), src_g, dst_g)
    want = O.canonical(O.bconv(src.astype(np.int32), src_g, dst_g), np.array(dst_g, np.uint32))
    np.testing.assert_array_equal(host(got), want)


@pytest.mark.parametrize("shape", [(8, 24), (10, 22), (2, 22), (1, 3), (16, 40)])
def test_bconv_cuda_core_matches_oracle(monkeypatch, shape):
    """The CUDA-core BConv (k_bconv, CK32_TC=0; the tcgen05 kernel is the
    default) equals the oracle."""
    monkeypatch.setenv("CK32_TC", "0")
    sc, dc = shape
    n, l, a = 65536, 40, 16
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=48))
    O = Oracle(n, l, a, 48)
    src_g = list(range(l - sc, l)) if sc <= 10 else [l + j for j in range(sc)]
    dst_g = list(range(dc))
    src = O.canonical(O.random_rows(Rng(sc * 100 + dc), np.array(src_g, np.uint32)), np.array(src_g, np.uint32))
    got = ckks.bconv(C, dev(src), src_g, dst_g)
    want = O.canonical(O.bconv(src.astype(np.int32), src_g, dst_g), np.array(dst_g, np.uint32))
    np.testing.assert_array_equal(host(got), want)
    C.close()


@pytest.fixture(params=["1", "2"])
def tc_env(monkeypatch, request):
    """Contexts created inside the test run BConv on the tcgen05 split-word
    GEMM (bconv_tc.cu; CK32_TC read at context creation): 1 = k_bconv_tc,
    2 = k_bconv_tc2 (the default)."""
    monkeypatch.setenv("CK32_TC", request.param)
    made = []

    def make(n, l, a, db=55):
        c = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db))
        made.append(c)
        return c
    yield make
    for c in made:
        c.close()


@pytest.mark.parametrize("mode", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("shape", [(8, 24), (10, 22), (1, 3), (16, 64)])
def test_bconv_fp64_pipe_matches_oracle(monkeypatch, mode, shape):
    """Exact BConv dot products on the FP64 pipe (CK32_BCONV_FP64, kernels.cu
    k_bconv_df / k_bconv_ws): bit-identical to the oracle for every row split,
    including 16 sources (the largest exactness bound)."""
    monkeypatch.setenv("CK32_BCONV_FP64", str(mode))
    n, l, a = 65536, 64, 16
    sc, dc = shape
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=48))
    O = _oracle(n, l, a, 48)
    src_g = list(range(l - sc, l)) if sc <= 10 else [l + j for j in range(sc)]
    dst_g = list(range(dc))
    src = O.canonical(O.random_rows(Rng(sc * 91 + dc + mode), np.array(src_g, np.uint32)), np.array(src_g, np.uint32))
    got = ckks.bconv(C, dev(src), src_g, dst_g)
    want = O.canonical(O.bconv(src.astype(np.int32), src_g, dst_g), np.array(dst_g, np.uint32))
    np.testing.assert_array_equal(host(got), want)
    C.close()


@pytest.mark.parametrize("n", [1024, 65536])
@pytest.mark.parametrize("shape", [(8, 24), (10, 22), (2, 22), (1, 3), (16, 40), (16, 64)])
def test_bconv_tensor_core_matches_oracle(tc_env, n, shape):
    sc, dc = shape
    l, a = 64, 16
    C = tc_env(n, l, a, 48)
    O = _oracle(n, l, a, 48)
    src_g = list(range(l - sc, l)) if sc <= 10 else [l + j for j in range(sc)]
    dst_g = list(range(dc))
    src = O.canonical(O.random_rows(Rng(sc * 77 + dc), np.array(src_g, np.uint32)), np.array(src_g, np.uint32))
    got = ckks.bconv(C, dev(src), src_g, dst_g)
    want = O.canonical(O.bconv(src.astype(np.int32), src_g, dst_g), np.array(dst_g, np.uint32))
    np.testing.assert_array_equal(host(got), want)


@pytest.mark.parametrize("level", [24, 17, 9, 4])
def test_mechanisms_tensor_core_bconv_match_oracle(tc_env, level):
    n, l, a, db = 4096, 24, 8, 55
    C = tc_env(n, l, a, db)
    O = _oracle(n, l, a, db)
    xb, xa, yb, ya, evk = O.synthetic(level, 31 + level)
    x, y = ct(np.stack([xb, xa]), level), ct(np.stack([yb, ya]), level)
    ob, oa = O.hmult(level, xb, xa, yb, ya, evk)
    got = host(ckks.hmult(C, x, y, ckks.EvaluationKey(dev(evk))).data)
    np.testing.assert_array_equal(got, np.stack([canon(O, ob, level - 2), canon(O, oa, level - 2)]))
    ob, oa = O.hrot(level, xb, xa, 5, evk)
    got = host(ckks.hrot(C, x, 5, ckks.EvaluationKey(dev(evk), ckks.ROTATION, 5)).data)
    np.testing.assert_array_equal(got, np.stack([canon(O, ob, level), canon(O, oa, level)]))


@pytest.mark.parametrize("r", [1, 3, -2, 1 << 14, 12345])
def test_automorphism_and_group_law(r):
    n, l, a = 65536, 4, 2
    C = ctx_for(n, l, a, 48)
    O = Oracle(n, l, a, 48)
    x = O.random_rows(Rng(r & 0xFFFF), O.gidx(l))
    p = ckks.Polynomial(dev(x), l)
    got = host(ckks.apply_automorphism(C, p, r).data)
    src = O.rotation_src_map(r)
    np.testing.assert_array_equal(got, x[:, src].astype(np.uint32))
    # rot_r then rot_-r is the identity (test_automorphism.cpp:29-39)
    back = ckks.apply_automorphism(C, ckks.apply_automorphism(C, p, r), -r)
    np.testing.assert_array_equal(host(back.data), x.astype(np.uint32))


# --------------------------------------------------------- small fixtures ----
@pytest.mark.parametrize("d", [pytest.param(d, id=d.name) for d in SMALL_DIRS])
def test_mechanisms_equal_reference_fixtures(d):
    fx = Fixture(d)
    C = ctx_for(fx.n, fx.l, fx.alpha, fx.db)
    np.testing.assert_array_equal(C.primes, fx.basis.primes)
    l, a = fx.l, fx.alpha
    u, v = fx.ct("ct_u"), fx.ct("ct_v")
    cu = ckks.Ciphertext(dev(Fixture.ct_rows(u)), u.scale, l)
    cv = ckks.Ciphertext(dev(Fixture.ct_rows(v)), v.scale, l)
    relin = ckks.EvaluationKey(dev(fx.evk("evk_relin").stacked()), ckks.RELIN)
    rot1 = ckks.EvaluationKey(dev(fx.evk("evk_rot1").stacked()), ckks.ROTATION, 1)
    rot3 = ckks.EvaluationKey(dev(fx.evk("evk_rot3").stacked()), ckks.ROTATION, 3)

    def eq(name, out):
        ref = fx.ct(name)
        assert out.level == ref.level, name
        assert out.scale == ref.scale, name
        assert out.pending_rescale == ref.pending_rescale, name
        np.testing.assert_array_equal(host(out.data), Fixture.ct_rows(ref), err_msg=name)

    eq("out_hmult", ckks.hmult(C, cu, cv, relin))
    eq("out_hrot1", ckks.hrot(C, cu, 1, rot1))
    eq("out_hrot3", ckks.hrot(C, cu, 3, rot3))
    eq("out_rescale", ckks.rescale(C, cu))
    eq("out_hadd", ckks.hadd(C, cu, cv))
    pv = fx.poly("pt_v")
    ptv = ckks.Plaintext(ckks.Polynomial(dev(pv.rows), l), Fraction(1 << fx.db), l)
    eq("out_pmult", ckks.pmult(C, cu, ptv))
    eq("out_padd", ckks.padd(C, cu, ptv))

    d_a = ckks.Polynomial(dev(u.a.rows), l)
    h = ckks.mod_up(C, d_a)
    hh = host(h.digits)
    for k in range(C.num_digits(l)):
        np.testing.assert_array_equal(hh[k], fx.poly(f"out_modup_d{k}").rows)
    v0, v1 = ckks.key_mult(C, h, relin)
    np.testing.assert_array_equal(host(v0.data), fx.poly("out_keymult_v0").rows)
    np.testing.assert_array_equal(host(v1.data), fx.poly("out_keymult_v1").rows)
    np.testing.assert_array_equal(host(ckks.mod_down(C, v0).data), fx.poly("out_moddown_v0").rows)
    c0, c1 = ckks.key_switch(C, d_a, relin)
    np.testing.assert_array_equal(host(c0.data), fx.poly("out_keyswitch_c0").rows)
    np.testing.assert_array_equal(host(c1.data), fx.poly("out_keyswitch_c1").rows)

    hr = ckks.hoisted_rotations(C, cu, [1, 3], [rot1, rot3])
    eq("out_hoisted_r1", hr[0])
    eq("out_hoisted_r3", hr[1])
    pts = [ckks.Plaintext(ckks.Polynomial(dev(fx.poly(f"pt_acc{i}").rows), l, a), Fraction(1 << fx.db), l)
           for i in range(3)]
    eq("out_hoisted_acc", ckks.hoisted_rotate_accumulate(C, cu, [0, 1, 3], pts, [None, rot1, rot3]))

    coeff = fx.poly("in_ntt_coeff")
    p = ckks.Polynomial(dev(coeff.rows), l, a, ckks.COEFFICIENT, False)
    np.testing.assert_array_equal(host(ckks.ntt_forward(C, p).data), fx.poly("out_ntt_coeff").rows)
    pb = ckks.Polynomial(dev(u.b.rows), l)
    np.testing.assert_array_equal(host(ckks.intt_inverse(C, pb).data), fx.poly("out_intt_ctub").rows)

    Cl = ctx_for(fx.n, fx.l, fx.alpha, fx.db, lazy=True)
    eq("out_hmult_lazy", ckks.hmult(Cl, cu, cv, relin))


# ---------------------------------------------------- full size (config 1/4) --
FULL_IDS = [f"{c[0]}:{c[2]}@{c[3]}@{c[4]}" for c in full_cases()]


@pytest.mark.parametrize("case", full_cases(), ids=FULL_IDS)
def test_full_size_matches_reference_hash(case):
    name, cfg, op, level, rot, h = case
    n, l, a, db = cfg["n"], cfg["l"], cfg["alpha"], cfg["delta_bits"]
    C = ctx_for(n, l, a, db, lazy=(op == "hmult_lazy"))
    O = _oracle(n, l, a, db)
    xb, xa, yb, ya, evk = O.synthetic(level, FULL["seed"])
    x = ct(np.stack([xb, xa]), level)
    y = ct(np.stack([yb, ya]), level)
    kind = ckks.ROTATION if op == "hrot" else ckks.RELIN
    K = ckks.EvaluationKey(dev(evk), kind, rot)
    if op in ("hmult", "hmult_lazy"):
        got = host(ckks.hmult(C, x, y, K).data)
    elif op == "hrot":
        got = host(ckks.hrot(C, x, rot, K).data)
    elif op == "rescale":
        got = host(ckks.rescale(C, x).data)
    elif op == "key_switch":
        c0, c1 = ckks.key_switch(C, ckks.Polynomial(dev(xa), level), K)
        got = np.concatenate([host(c0.data), host(c1.data)])
    elif op == "mod_up":
        got = host(ckks.mod_up(C, ckks.Polynomial(dev(xa), level)).digits)
    elif op == "ntt":
        got = host(ckks.ntt_forward(C, ckks.Polynomial(dev(xb), level, 0, ckks.COEFFICIENT, False)).data)
    elif op == "intt":
        got = host(ckks.intt_inverse(C, ckks.Polynomial(dev(xb), level)).data)
    else:
        raise AssertionError(op)
    assert sha(got) == h


_OR = {}


def _oracle(n, l, a, db):
    if (n, l, a, db) not in _OR:
        _OR[(n, l, a, db)] = Oracle(n, l, a, db)
    return _OR[(n, l, a, db)]


# ------------------------------------------------- oracle sweeps / batching --
@pytest.mark.parametrize("level", [24, 23, 17, 9, 5, 4])
def test_hmult_hrot_oracle_sweep_mid_size(level):
    n, l, a, db = 4096, 24, 8, 55
    C = ctx_for(n, l, a, db)
    O = _oracle(n, l, a, db)
    xb, xa, yb, ya, evk = O.synthetic(level, 99 + level)
    x, y = ct(np.stack([xb, xa]), level), ct(np.stack([yb, ya]), level)
    ob, oa = O.hmult(level, xb, xa, yb, ya, evk)
    got = host(ckks.hmult(C, x, y, ckks.EvaluationKey(dev(evk))).data)
    np.testing.assert_array_equal(got, np.stack([canon(O, ob, level - 2), canon(O, oa, level - 2)]))
    for r in (1, -7, n // 4):
        ob, oa = O.hrot(level, xb, xa, r, evk)
        got = host(ckks.hrot(C, x, r, ckks.EvaluationKey(dev(evk), ckks.ROTATION, r)).data)
        np.testing.assert_array_equal(got, np.stack([canon(O, ob, level), canon(O, oa, level)]))


@pytest.mark.parametrize("level", [54, 41, 28, 15, 4])
def test_reference_default_params_match_oracle(level):
    """The reference's default CkksParams (ckks.hpp:46-54: l=54, alpha=14,
    delta 2^48 -> D=4 digits, a ragged 12-row last digit, 14-wide BConv
    sources and the 16-row merged ModDown) at N=4096, HMult and HRot vs the
    oracle, batched over 2 ciphertexts."""
    n, l, a, db = 4096, 54, 14, 48
    C = ctx_for(n, l, a, db)
    O = _oracle(n, l, a, db)
    xs, ys, want_m, want_r = [], [], [], []
    evk = None
    for b in range(2):
        xb, xa, yb, ya, evk_b = O.synthetic(level, 4242 + 10 * level + b)
        evk = evk_b if evk is None else evk  # one key for the whole batch
        xs.append(np.stack([xb, xa]))
        ys.append(np.stack([yb, ya]))
        if level >= 4:
            ob, oa = O.hmult(level, xb, xa, yb, ya, evk)
            want_m.append(np.stack([canon(O, ob, level - 2), canon(O, oa, level - 2)]))
        ob, oa = O.hrot(level, xb, xa, 3, evk)
        want_r.append(np.stack([canon(O, ob, level), canon(O, oa, level)]))
    K = ckks.EvaluationKey(dev(evk))
    X = ckks.Ciphertext(dev(np.stack(xs)), Fraction(1 << db), level)
    Y = ckks.Ciphertext(dev(np.stack(ys)), Fraction(1 << db), level)
    got = host(ckks.hmult(C, X, Y, K).data)
    np.testing.assert_array_equal(got, np.stack(want_m))
    got = host(ckks.hrot(C, X, 3, ckks.EvaluationKey(K.data, ckks.ROTATION, 3)).data)
    np.testing.assert_array_equal(got, np.stack(want_r))


def test_batched_equals_unbatched():
    n, l, a, db = 65536, 24, 8, 55
    C = ctx_for(n, l, a, db)
    O = _oracle(n, l, a, db)
    B = 3
    xs, ys = [], []
    for b in range(B):
        xb, xa, yb, ya, evk = O.synthetic(24, 500 + b)
        xs.append(np.stack([xb, xa]))
        ys.append(np.stack([yb, ya]))
    K = ckks.EvaluationKey(dev(evk))
    KR = ckks.EvaluationKey(K.data, ckks.ROTATION, 1)
    X = ckks.Ciphertext(dev(np.stack(xs)), Fraction(1 << 55), 24)
    Y = ckks.Ciphertext(dev(np.stack(ys)), Fraction(1 << 55), 24)
    hm = host(ckks.hmult(C, X, Y, K).data)
    hr = host(ckks.hrot(C, X, 1, KR).data)
    for b in range(B):
        one = host(ckks.hmult(C, ct(xs[b], 24), ct(ys[b], 24), K).data)
        np.testing.assert_array_equal(hm[b], one)
        one = host(ckks.hrot(C, ct(xs[b], 24), 1, KR).data)
        np.testing.assert_array_equal(hr[b], one)


@pytest.mark.parametrize("km", ["8", "12", "13", "14", "15", "16"])
@pytest.mark.parametrize("level,B", [(24, 6), (9, 8)])
def test_batched_keymult_variants_equal_unbatched(km, level, B):
    """The fused row pass + KeyMult variants at batch B >= 4 (CK32_KM=12:
    k_row_keymult8b, four batch items per CTA sharing the row's key slice and
    twiddles; B = 6 leaves two idle warps in the last item group): every
    ciphertext of the batched HMult / HRot equals its B = 1 result, and the
    first one equals the oracle (fresh subprocess: CK32_KM is read once)."""
    import subprocess
    import sys
    from pathlib import Path

    code = f'''
import sys, numpy as np, torch
sys.path[:0] = {[str(Path(__file__).resolve().parent.parent), str(Path(__file__).resolve().parent.parent / "oracle")]!r}
from fractions import Fraction
from paper_2407_13055_b200 import ckks
from pyoracle import Oracle, Rng
n, l, a, db, level, B = 1 << 16, 24, 8, 55, {level}, {B}
O = Oracle(n, l, a, db)
dev = lambda v: torch.from_numpy(np.ascontiguousarray(v.astype(np.int32))).cuda()
C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db))
xs, ys = [], []
for b in range(B):
    xb, xa, yb, ya, evk = O.synthetic(level, 700 + b)
    xs.append(np.stack([xb, xa])); ys.append(np.stack([yb, ya]))
K = ckks.EvaluationKey(dev(evk)); KR = ckks.EvaluationKey(K.data, ckks.ROTATION, 1)
ct = lambda v: ckks.Ciphertext(dev(v), Fraction(1 << db), level)
hm = ckks.hmult(C, ct(np.stack(xs)), ct(np.stack(ys)), K).data.cpu().numpy().astype(np.uint32)
hr = ckks.hrot(C, ct(np.stack(xs)), 1, KR).data.cpu().numpy().astype(np.uint32)
for b in range(B):
    assert np.array_equal(hm[b], ckks.hmult(C, ct(xs[b]), ct(ys[b]), K).data.cpu().numpy().astype(np.uint32)), b
    assert np.array_equal(hr[b], ckks.hrot(C, ct(xs[b]), 1, KR).data.cpu().numpy().astype(np.uint32)), b
ob, oa = O.hmult(level, xs[0][0], xs[0][1], ys[0][0], ys[0][1], evk)
assert np.array_equal(hm[0], np.stack([O.canonical(ob, O.gidx(level - 2)), O.canonical(oa, O.gidx(level - 2))]))
print("batched ok")
'''
    env = dict(__import__("os").environ, CK32_KM=km)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0 and "batched ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("chunk,depth", [(2, 2), (3, 3), (8, 2)])
def test_host_pipeline_equals_direct(chunk, depth):
    """pipeline.HostPipeline (chunked H2D / compute / D2H on separate streams,
    used by bench.py's e2e leg) returns exactly the direct batched results,
    also across back-to-back runs that overlap."""
    from paper_2407_13055_b200.pipeline import HostPipeline

    n, l, a, db, B, level = 4096, 24, 8, 55, 7, 24
    C = ctx_for(n, l, a, db)
    O = _oracle(n, l, a, db)
    xs, ys = [], []
    for b in range(B):
        xb, xa, yb, ya, evk = O.synthetic(level, 700 + b)
        xs.append(np.stack([xb, xa]))
        ys.append(np.stack([yb, ya]))
    K = ckks.EvaluationKey(dev(evk))
    KR = ckks.EvaluationKey(K.data, ckks.ROTATION, 1)
    s = Fraction(1 << 55)
    X = ckks.Ciphertext(dev(np.stack(xs)), s, level)
    Y = ckks.Ciphertext(dev(np.stack(ys)), s, level)
    want1 = host(ckks.hmult(C, X, Y, K).data)
    want2 = host(ckks.hrot(C, X, 1, KR).data)
    hx, hy = X.data.cpu().pin_memory(), Y.data.cpu().pin_memory()
    ho1 = torch.zeros((B, 2, level - 2, n), dtype=torch.int32).pin_memory()
    ho2 = torch.zeros((B, 2, level, n), dtype=torch.int32).pin_memory()
    pipe = HostPipeline(torch.device("cuda", 0), chunk=chunk, depth=depth)

    def fn(d):
        cx = ckks.Ciphertext(d[0], s, level)
        return ckks.hmult(C, cx, ckks.Ciphertext(d[1], s, level), K).data, ckks.hrot(C, cx, 1, KR).data

    for _ in range(3):
        ev = pipe.run([hx, hy], fn, [ho1, ho2])
    ev.synchronize()
    np.testing.assert_array_equal(ho1.numpy().astype(np.uint32), want1)
    np.testing.assert_array_equal(ho2.numpy().astype(np.uint32), want2)
    with pytest.raises(ValueError):
        pipe.run([X.data, hy], fn, [ho1, ho2])  # device tensor where a pinned host one is required

    # results written into the pipeline's own per-slot buffers (the evaluator's out= arguments)
    def fn_inplace(d, o):
        cx = ckks.Ciphertext(d[0], s, level)
        return (ckks.hmult(C, cx, ckks.Ciphertext(d[1], s, level), K, out=o[0]).data,
                ckks.hrot(C, cx, 1, KR, out=o[1]).data)

    ho1.zero_()
    ho2.zero_()
    for _ in range(3):
        ev = pipe.run([hx, hy], fn_inplace, [ho1, ho2], outputs_in_place=True)
    ev.synchronize()
    np.testing.assert_array_equal(ho1.numpy().astype(np.uint32), want1)
    np.testing.assert_array_equal(ho2.numpy().astype(np.uint32), want2)
    with pytest.raises(ValueError):  # out= of the wrong shape
        ckks.hmult(C, X, Y, K, out=torch.empty((B, 2, level, n), dtype=torch.int32, device="cuda"))


def test_captured_step_replays_bit_exactly():
    """pipeline.CapturedStep: HMult + HRot captured in a CUDA graph, replayed
    on fresh inputs copied into the static buffers, equals eager calls."""
    from paper_2407_13055_b200.pipeline import CapturedStep

    n, l, a, db, level = 4096, 24, 8, 55, 24
    C = ctx_for(n, l, a, db)
    O = _oracle(n, l, a, db)
    xb, xa, yb, ya, evk = O.synthetic(level, 808)
    K = ckks.EvaluationKey(dev(evk))
    KR = ckks.EvaluationKey(K.data, ckks.ROTATION, 1)
    s = Fraction(1 << 55)
    X = ckks.Ciphertext(dev(np.stack([xb, xa])), s, level)
    Y = ckks.Ciphertext(dev(np.stack([yb, ya])), s, level)
    step = CapturedStep(torch.device("cuda", 0), lambda: (ckks.hmult(C, X, Y, K).data, ckks.hrot(C, X, 1, KR).data))
    for seed in (809, 810):
        nb, na, mb, ma, _ = O.synthetic(level, seed)
        X.data.copy_(dev(np.stack([nb, na])))
        Y.data.copy_(dev(np.stack([mb, ma])))
        m, r = step.replay()
        want_m = host(ckks.hmult(C, X, Y, K).data)
        want_r = host(ckks.hrot(C, X, 1, KR).data)
        np.testing.assert_array_equal(host(m), want_m)
        np.testing.assert_array_equal(host(r), want_r)


def test_counters_follow_reference_profile():
    # HMult at l=24: ntt 116, intt 44, bconv 5, keymult 3; HRot: ntt 120, intt 40
    n, l, a, db = 1024, 24, 8, 55
    C = ctx_for(n, l, a, db)
    O = _oracle(n, l, a, db)
    xb, xa, yb, ya, evk = O.synthetic(24, 1)
    x, y = ct(np.stack([xb, xa]), 24), ct(np.stack([yb, ya]), 24)
    C.reset_counters()
    ckks.hmult(C, x, y, ckks.EvaluationKey(dev(evk)))
    c = C.counters()
    assert (c["modup"], c["moddown"], c["ntt"], c["intt"], c["keymult"], c["bconv"]) == (1, 1, 116, 44, 3, 5)
    C.reset_counters()
    ckks.hrot(C, x, 1, ckks.EvaluationKey(dev(evk), ckks.ROTATION, 1))
    c = C.counters()
    assert (c["modup"], c["moddown"], c["ntt"], c["intt"], c["keymult"], c["bconv"]) == (1, 1, 120, 40, 3, 5)


def test_errors_mirror_reference():
    n, l, a, db = 1024, 24, 8, 55
    C = ctx_for(n, l, a, db)
    O = _oracle(n, l, a, db)
    xb, xa, yb, ya, evk = O.synthetic(4, 2)
    x = ct(np.stack([xb, xa]), 4)
    K = ckks.EvaluationKey(dev(evk))
    with pytest.raises(ValueError):  # rotation key for hmult
        ckks.hmult(C, x, x, ckks.EvaluationKey(K.data, ckks.ROTATION, 1))
    with pytest.raises(ValueError):  # wrong rotation amount
        ckks.hrot(C, x, 2, ckks.EvaluationKey(K.data, ckks.ROTATION, 1))
    x2 = ct(np.stack([xb[:2], xa[:2]]), 2)
    with pytest.raises(ValueError):  # level exhausted (ckks.cpp:815)
        ckks.hmult(C, x2, x2, K)
    with pytest.raises(ValueError):
        ckks.rescale(C, x2)
    bad = ckks.Ciphertext(x.data, x.scale * Fraction(1025, 1024), 4)
    with pytest.raises(ValueError):  # scale mismatch beyond 2^-40 (ckks.cpp:131-136)
        ckks.hadd(C, x, bad)
    p = ckks.Polynomial(dev(xb), 4)
    with pytest.raises(ValueError):  # domain discipline (ntt.cpp:290-292)
        ckks.ntt_forward(C, p)
    with pytest.raises(ValueError):
        ckks.CkksContext(ckks.CkksParams(n=1000, l=4, alpha=2))
    # mod_switch argument checks (bconv.cpp:180-197)
    pe = ckks.Polynomial(dev(xb), 4)
    with pytest.raises(ValueError):  # rows do not match the table source
        ckks.mod_switch(C, pe, [0, 1], 2)
    with pytest.raises(ValueError):  # coefficient-domain input
        ckks.mod_switch(C, ckks.Polynomial(dev(xb), 4, 0, ckks.COEFFICIENT, False), [0, 1, 2, 3], 2)
    with pytest.raises(ValueError):  # destination wider than the basis
        ckks.mod_switch(C, pe, [0, 1, 2, 3], l + 1)
    # decode checks (ckks.cpp:322)
    with pytest.raises(ValueError):
        ckks.decode(C, ckks.Plaintext(ckks.Polynomial(dev(xb), 4, 0, ckks.COEFFICIENT, False), Fraction(1 << 55), 4))


def test_lazy_then_rescale_equals_merged_ledger():
    # merged and lazy paths agree on level/scale after the deferred rescale (test_ckks.cpp:320-362)
    n, l, a, db = 1024, 8, 2, 48
    Cm, Cl = ctx_for(n, l, a, db), ctx_for(n, l, a, db, lazy=True)
    O = _oracle(n, l, a, db)
    xb, xa, yb, ya, evk = O.synthetic(8, 3)
    s = Fraction(1 << 48)
    x, y = ct(np.stack([xb, xa]), 8, s), ct(np.stack([yb, ya]), 8, s)
    K = ckks.EvaluationKey(dev(evk))
    pm = ckks.hmult(Cm, x, y, K)
    pl = ckks.hmult(Cl, x, y, K)
    assert pl.pending_rescale and pl.level == 8
    pr = ckks.rescale(Cl, pl)
    assert (pm.level, pm.scale) == (pr.level, pr.scale)


def test_cpp_mirror_drop_in(tmp_path):
    """The header-only C++ mirror (ckks32_b200.hpp) over the C ABI, driven by a
    C++ program the way the reference's tests drive ckks.hpp."""
    import subprocess
    from pathlib import Path

    exe = Path(__file__).resolve().parent.parent / "paper_2407_13055_b200" / "_lib" / "test_cpp_api"
    if not exe.exists():
        subprocess.run(["make", "-C", str(exe.parent.parent), "cpp_test"], check=True, capture_output=True)
    n, l, a, db, level = 4096, 12, 4, 55, 10
    O = _oracle(n, l, a, db)
    xb, xa, yb, ya, evk = O.synthetic(level, 77)
    np.stack([xb, xa]).astype("<u4").tofile(tmp_path / "x.bin")
    np.stack([yb, ya]).astype("<u4").tofile(tmp_path / "y.bin")
    evk.astype("<u4").tofile(tmp_path / "evk.bin")
    r = subprocess.run([str(exe), str(tmp_path), str(n), str(l), str(a), str(level)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cpp api ok" in r.stdout
    ob, oa = O.hmult(level, xb, xa, yb, ya, evk)
    got = np.fromfile(tmp_path / "out_hmult.bin", dtype="<u4").reshape(2, level - 2, n)
    np.testing.assert_array_equal(got, np.stack([canon(O, ob, level - 2), canon(O, oa, level - 2)]))
    rb, ra = O.hrot(level, xb, xa, 1, evk)
    got = np.fromfile(tmp_path / "out_hrot.bin", dtype="<u4").reshape(2, level, n)
    np.testing.assert_array_equal(got, np.stack([canon(O, rb, level), canon(O, ra, level)]))
    # the mirror's hoisted_rotate_accumulate (pt = Montgomery one, P-extended, r = 1)
    g = O.gidx(level, a)
    one = np.repeat(np.array([(1 << 32) % int(q) for q in O.primes[g]], np.int64)[:, None], n, 1)
    ab, aa = O.hoisted_accumulate(level, xb, xa, [1], [one], [evk])
    got = np.fromfile(tmp_path / "out_acc.bin", dtype="<u4").reshape(2, level, n)
    np.testing.assert_array_equal(got, np.stack([canon(O, ab, level), canon(O, aa, level)]))


def test_cpp_mirror_keys_with_std_mt19937_64(tmp_path):
    """keygen / evk_gen / encode / encrypt of the C++ mirror take the
    caller's std::mt19937_64 (ckks.hpp:155-167) and reproduce the reference's
    own fixtures bit for bit (sk.s, relin / rot 1 / rot 3 keys, ct_u, ct_v of
    tests/golden)."""
    import subprocess
    from pathlib import Path

    from golden_util import SMALL_DIRS, SMALL_SEEDS, Fixture, parse_small_name

    exe = Path(__file__).resolve().parent.parent / "paper_2407_13055_b200" / "_lib" / "test_cpp_api"
    if not exe.exists():
        subprocess.run(["make", "-C", str(exe.parent.parent), "cpp_test"], check=True, capture_output=True)
    for d in SMALL_DIRS:
        F = Fixture(d)
        n, l, a = parse_small_name(d)
        r = subprocess.run([str(exe), "keys", str(tmp_path), str(SMALL_SEEDS[(n, l, a)]), str(n), str(l), str(a),
                            str(F.db)], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "cpp keys ok" in r.stdout, r.stdout + r.stderr
        sk = np.fromfile(tmp_path / "sk_rows.bin", dtype="<u4").reshape(l + a, n)
        np.testing.assert_array_equal(sk, F.poly("sk").rows)
        for name in ("evk_relin", "evk_rot1", "evk_rot3"):
            want = F.evk(name).stacked()
            got = np.fromfile(tmp_path / f"{name}.bin", dtype="<u4").reshape(want.shape)
            np.testing.assert_array_equal(got, want, err_msg=f"{d.name} {name}")
        np.testing.assert_array_equal(np.fromfile(tmp_path / "pt_v.bin", dtype="<u4").reshape(l, n),
                                      F.poly("pt_v").rows, err_msg=f"{d.name} pt_v")
        for name in ("ct_u", "ct_v"):
            got = np.fromfile(tmp_path / f"{name}.bin", dtype="<u4").reshape(2, l, n)
            want = Fixture.ct_rows(F.ct(name))
            np.testing.assert_array_equal(got[1], want[1], err_msg=f"{d.name} {name}.a")
            np.testing.assert_array_equal(got[0], want[0], err_msg=f"{d.name} {name}.b")


# ------------------------------------------------------------- mod_switch --
@pytest.mark.parametrize("n", [16, 32, 64, 65536])
def test_mod_switch_error_characterization(n):
    """test_bconv.cpp:147-190 on the GPU: P basis -> Q prefix; after INTT the
    output equals (exact + e P) mod q with 0 <= e < alpha (alpha = 2)."""
    l, a = 2, 2
    C = ctx_for(n, l, a, 48)
    O = _oracle(n, l, a, 48)
    P = [int(p) for p in O.primes[l:]]
    rng = np.random.default_rng(113 + n)
    coeffs = np.stack([rng.integers(0, p, n) for p in P]).astype(np.uint32)
    src_g = [l, l + 1]
    poly = ckks.ntt_forward(C, ckks.Polynomial(dev(coeffs), 0, a, ckks.COEFFICIENT, False))
    out = ckks.mod_switch(C, poly, src_g, 2, 0)
    assert out.domain == ckks.EVALUATION and out.mont
    back = host(ckks.intt_inverse(C, out).data).astype(object)
    Pprod = P[0] * P[1]
    # CRT of the source residues (exact integer in [0, P))
    inv = [pow(Pprod // p, -1, p) for p in P]
    exact = [(int(coeffs[0, j]) * inv[0] * (Pprod // P[0]) + int(coeffs[1, j]) * inv[1] * (Pprod // P[1])) % Pprod
             for j in range(n)]
    for i in range(2):
        q = int(O.primes[i])
        for j in range(n):
            assert int(back[i, j]) in {(exact[j] + e * Pprod) % q for e in range(a)}


def test_mod_switch_small_constant_is_exact():
    """test_bconv.cpp:192-208: a small constant polynomial switches exactly."""
    n, l, a = 16, 2, 1
    C = ctx_for(n, l, a, 48)
    coeffs = np.arange(1, n + 1, dtype=np.uint32)[None, :]
    poly = ckks.ntt_forward(C, ckks.Polynomial(dev(coeffs), 0, a, ckks.COEFFICIENT, False))
    out = ckks.intt_inverse(C, ckks.mod_switch(C, poly, [l], 2, 0))
    np.testing.assert_array_equal(host(out.data), np.stack([np.arange(1, n + 1)] * 2).astype(np.uint32))


@pytest.mark.parametrize("n", [1024, 65536])
def test_mod_switch_matches_oracle_composition(n):
    """bconv.cpp:176-213 = inverse_row(part1) -> bconv_part2 -> forward_row,
    composed from the oracle's pinned INTT / BConv / NTT."""
    l, a = 12, 4
    C = ctx_for(n, l, a, 48)
    O = _oracle(n, l, a, 48)
    src_g = np.array([l + j for j in range(a)], np.uint32)
    dst_g = np.array(list(range(6)) + [l, l + 1], np.uint32)
    x = O.random_rows(Rng(n + 5), src_g)  # canonical evaluation-domain residues
    out = ckks.mod_switch(C, ckks.Polynomial(dev(x), 0, a), list(src_g), 6, 2)
    part1 = [int(v) for v in O.bconv_part1(src_g)]
    coef = O.canonical(O.intt(x, src_g, part1), src_g)
    conv = O.bconv(coef.astype(np.int32), list(src_g), list(dst_g))
    want = O.canonical(O.ntt_fwd(conv, dst_g), dst_g)
    np.testing.assert_array_equal(host(out.data), want)


# ------------------------------------------- element-wise (a5), automorphism (a13)
@pytest.mark.parametrize("n", [1024, 65536])
@pytest.mark.parametrize("q_rows,p_rows", [(8, 0), (5, 3), (8, 3), (1, 1)])
def test_elementwise_ops_match_oracle(n, q_rows, p_rows):
    """ew_add / ew_sub / ew_mul / ew_mul_const and the in-place add / sub
    (poly.cpp:121-205) over Q-prefix and P-extended polynomials, canonical
    residues equal to the oracle's."""
    l, a = 8, 3
    C = ctx_for(n, l, a)
    O = Oracle(n, l, a, 55)
    rng = Rng(17 * n + q_rows)
    g = O.gidx(q_rows, p_rows)
    x, y = O.random_rows(rng, g), O.random_rows(rng, g)
    X = ckks.Polynomial(dev(x), q_rows, p_rows)
    Y = ckks.Polynomial(dev(y), q_rows, p_rows)
    for op, fn in ((0, ckks.ew_add), (1, ckks.ew_sub), (2, ckks.ew_mul)):
        got = host(fn(C, X, Y).data)
        np.testing.assert_array_equal(got, O.canonical(O.ew(op, x, y, g), g), err_msg=f"op {op}")
    k = [int(v) for v in (np.arange(1, len(g) + 1) * 7919 + 3) % O.primes[g]]
    got = host(ckks.ew_mul_const(C, X, k).data)
    np.testing.assert_array_equal(got, O.canonical(O.ew(3, x, None, g, k), g))
    Z = X.clone()
    ckks.ew_add_inplace(C, Z, Y)
    np.testing.assert_array_equal(host(Z.data), O.canonical(O.ew(0, x, y, g), g))
    ckks.ew_sub_inplace(C, Z, Y)
    np.testing.assert_array_equal(host(Z.data), x.astype(np.uint32))
    if p_rows:  # basis prefix mismatch (check_binary, poly.cpp:115-119)
        with pytest.raises(ValueError):
            ckks.ew_add(C, X, ckks.Polynomial(Y.data, q_rows + p_rows, 0))


@pytest.mark.parametrize("n", [16, 1024, 65536])
@pytest.mark.parametrize("which", ["r1", "r-3", "r5", "r_n/4", "conj"])
def test_automorphism_both_domains_match_oracle(n, which):
    """apply_automorphism (automorphism.cpp:76-100): the evaluation-domain
    gather and the coefficient-domain signed permutation for rotation and
    conjugation maps, over a P-extended polynomial; and the coefficient
    variant commutes with the NTT (test_automorphism.cpp:71-96)."""
    l, a = 4, 2
    C = ctx_for(n, l, a, 48)
    O = Oracle(n, l, a, 48)
    r = {"r1": 1, "r-3": -3, "r5": 5, "r_n/4": n // 4}.get(which, 0)
    gal = 2 * n - 1 if which == "conj" else ckks.galois_for_rotation(n, r)
    g = O.gidx(l, a)
    x = O.random_rows(Rng(n + 99), g)
    for coeff in (False, True):
        P = ckks.Polynomial(dev(x), l, a, ckks.COEFFICIENT if coeff else ckks.EVALUATION, not coeff)
        got = host(ckks.apply_automorphism(C, P, r, galois=gal).data)
        np.testing.assert_array_equal(got, O.canonical(O.automorphism(x, gal, coeff), g), err_msg=f"coeff={coeff}")
        if which != "conj" and not coeff:  # the rotation entry point agrees with the Galois one
            np.testing.assert_array_equal(host(ckks.apply_automorphism(C, P, r).data), got)
    # commutation: NTT(phi_coeff(x)) == phi_eval(NTT(x))
    A = ckks.Polynomial(dev(x), l, a, ckks.COEFFICIENT, False)
    lhs = ckks.ntt_forward(C, ckks.apply_automorphism(C, A, r, galois=gal))
    rhs = ckks.apply_automorphism(C, ckks.ntt_forward(C, A.clone()), r, galois=gal)
    np.testing.assert_array_equal(host(lhs.data), host(rhs.data))


# ------------------------------------------------------- wire formats (f2) ----
@pytest.mark.parametrize("d", [pytest.param(d, id=d.name) for d in SMALL_DIRS])
def test_wire_formats_through_the_c_abi_are_byte_exact(d):
    """Ciphertexts, keys, polynomials and the basis read by the C ABI's
    deserialisers straight into device memory, HMult / HRot / key switching
    on the GPU, results written by the C ABI's serialisers: every blob is
    byte-identical to the one the reference wrote (ckks.cpp:1090-1154,
    poly.cpp:295-352, rns.cpp:168-216)."""
    fx = Fixture(d)
    C = ctx_for(fx.n, fx.l, fx.alpha, fx.db)
    blob = lambda name: (d / f"{name}.bin").read_bytes()
    assert ckks.serialize_basis(C) == blob("basis")
    cu, cv = ckks.deserialize_ciphertext(C, blob("ct_u")), ckks.deserialize_ciphertext(C, blob("ct_v"))
    assert ckks.serialize_ciphertext(C, cu) == blob("ct_u")
    relin = ckks.deserialize_evk(C, blob("evk_relin"))
    rot1 = ckks.deserialize_evk(C, blob("evk_rot1"))
    assert (relin.kind, rot1.kind, rot1.rotation) == (ckks.RELIN, ckks.ROTATION, 1)
    assert ckks.serialize_evk(C, relin) == blob("evk_relin")
    assert ckks.serialize_evk(C, rot1) == blob("evk_rot1")
    assert ckks.serialize_ciphertext(C, ckks.hmult(C, cu, cv, relin)) == blob("out_hmult")
    assert ckks.serialize_ciphertext(C, ckks.hrot(C, cu, 1, rot1)) == blob("out_hrot1")
    assert ckks.serialize_ciphertext(C, ckks.rescale(C, cu)) == blob("out_rescale")
    Cl = ctx_for(fx.n, fx.l, fx.alpha, fx.db, lazy=True)
    out_lazy = ckks.hmult(Cl, cu, cv, relin)
    assert out_lazy.pending_rescale and ckks.serialize_ciphertext(Cl, out_lazy) == blob("out_hmult_lazy")
    d_a = ckks.Polynomial(cu.data[1].contiguous(), fx.l)
    c0, c1 = ckks.key_switch(C, d_a, relin)
    assert ckks.serialize_poly(C, c0) == blob("out_keyswitch_c0")
    assert ckks.serialize_poly(C, c1) == blob("out_keyswitch_c1")
    p = ckks.deserialize_poly(C, blob("in_ntt_coeff"))
    assert (p.q_count, p.p_count, p.domain, p.mont) == (fx.l, fx.alpha, ckks.COEFFICIENT, False)
    assert ckks.serialize_poly(C, ckks.ntt_forward(C, p)) == blob("out_ntt_coeff")
    sk = ckks.deserialize_poly(C, blob("sk"))
    assert ckks.serialize_poly(C, sk) == blob("sk")


@pytest.mark.parametrize("d", [pytest.param(SMALL_DIRS[0], id=SMALL_DIRS[0].name)])
def test_wire_readers_reject_like_the_reference(d):
    """Truncation, bad magic, basis-hash and shape mismatches are errors of
    the reference's classes (runtime_error for polynomials, invalid_argument
    for ciphertext / key headers); non-canonical residues are rejected."""
    fx = Fixture(d)
    C = ctx_for(fx.n, fx.l, fx.alpha, fx.db)
    ct = (d / "ct_u.bin").read_bytes()
    pol = (d / "sk.bin").read_bytes()
    with pytest.raises(ValueError, match="header"):
        ckks.deserialize_ciphertext(C, b"XXXX" + ct[4:])
    with pytest.raises(ValueError, match="truncated"):
        ckks.deserialize_ciphertext(C, ct[: len(ct) // 2])
    with pytest.raises(RuntimeError, match="magic"):
        ckks.deserialize_poly(C, b"XXXX" + pol[4:])
    with pytest.raises(RuntimeError, match="truncated"):
        ckks.deserialize_poly(C, pol[:-4])
    bad_hash = bytearray(pol)
    bad_hash[24] ^= 1
    with pytest.raises(RuntimeError, match="hash"):
        ckks.deserialize_poly(C, bytes(bad_hash))
    big = bytearray(pol)
    big[32:36] = (0xFFFFFFF0).to_bytes(4, "little")
    with pytest.raises(RuntimeError, match="range"):
        ckks.deserialize_poly(C, bytes(big))
    with pytest.raises(ValueError):
        ckks.deserialize_evk(C, (d / "ct_u.bin").read_bytes())


@pytest.mark.parametrize("level,r", [(24, 1), (17, -3), (8, 1 << 14), (3, 5)])
def test_fused_hrot_tail_matches_oracle(monkeypatch, level, r):
    """The opt-in HRot path with combine + b + automorphism fused into the
    ModDown forward row pass (CK32_FUSED_TAIL=1, shared-memory-staged
    32-block stores) equals the oracle, batched (B = 2)."""
    monkeypatch.setenv("CK32_FUSED_TAIL", "1")
    n, l, a, db, B = 1 << 16, 24, 8, 55, 2
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db))
    O = _oracle(n, l, a, db)
    xs, want = [], []
    evk = O.synthetic(level, 499 + level)[4]  # one key for the batch
    for b in range(B):
        xb, xa = O.synthetic(level, 500 + 7 * b + level)[:2]
        xs.append(np.stack([xb, xa]))
        ob, oa = O.hrot(level, xb, xa, r, evk)
        want.append(np.stack([canon(O, ob, level), canon(O, oa, level)]))
    K = ckks.EvaluationKey(dev(evk), ckks.ROTATION, r)
    got = host(ckks.hrot(C, ckks.Ciphertext(dev(np.stack(xs)), Fraction(1 << db), level), r, K).data)
    np.testing.assert_array_equal(got, np.stack(want))
    C.close()


@pytest.mark.parametrize("level", [24, 13, 4])
def test_keymult_fused_intt_pass_a_matches_oracle(monkeypatch, level):
    """The opt-in path with the following switch's INTT pass A run in the
    KeyMult epilogue (CK32_KM_INTT=1, read once per process: run in a fresh
    subprocess) -- merged and lazy HMult and HRot equal the oracle."""
    import subprocess
    import sys
    from pathlib import Path

    code = f'''
import sys, numpy as np, torch
sys.path[:0] = {[str(Path(__file__).resolve().parent.parent), str(Path(__file__).resolve().parent.parent / "oracle")]!r}
from fractions import Fraction
from paper_2407_13055_b200 import ckks
from pyoracle import Oracle
n, l, a, db, level = 1 << 16, 24, 8, 55, {level}
O = Oracle(n, l, a, db)
xb, xa, yb, ya, evk = O.synthetic(level, 777 + level)
dev = lambda v: torch.from_numpy(np.ascontiguousarray(v.astype(np.int32))).cuda()
for lazy in (False, True):
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db, lazy_rescale=lazy))
    x = ckks.Ciphertext(dev(np.stack([xb, xa])), Fraction(1 << db), level)
    y = ckks.Ciphertext(dev(np.stack([yb, ya])), Fraction(1 << db), level)
    got = ckks.hmult(C, x, y, ckks.EvaluationKey(dev(evk))).data.cpu().numpy().astype(np.uint32)
    ob, oa = O.hmult(level, xb, xa, yb, ya, evk, lazy=lazy)
    lo = level if lazy else level - 2
    assert np.array_equal(got, np.stack([O.canonical(ob, O.gidx(lo)), O.canonical(oa, O.gidx(lo))])), lazy
    if not lazy:
        got = ckks.hrot(C, x, 3, ckks.EvaluationKey(dev(evk), ckks.ROTATION, 3)).data.cpu().numpy().astype(np.uint32)
        ob, oa = O.hrot(level, xb, xa, 3, evk)
        assert np.array_equal(got, np.stack([O.canonical(ob, O.gidx(level)), O.canonical(oa, O.gidx(level))]))
    C.close()
print("fused-intt ok")
'''
    env = dict(__import__("os").environ, CK32_KM_INTT="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and "fused-intt ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("level", [24, 7])
@pytest.mark.parametrize("variant", ["CK32_ROW8=1", "CK32_KM=7", "CK32_KM=9", "CK32_KM=10", "CK32_KM=11", "CK32_TC=0",
                                     "CK32_COL=3", "CK32_COL=4", "CK32_COL=5", "CK32_KM=12", "CK32_KM=13", "CK32_KM=14", "CK32_KM=15", "CK32_KM=16",
                                     "CK32_TAIL_GATHER=1"])
def test_variant_paths_match_oracle(level, variant):
    """Opt-in kernel variants (env switches read once per process: a fresh
    subprocess each) -- CK32_ROW8=1: the plain row passes as k_row8 (8
    coefficients per thread); CK32_KM=7/9/10/11: the fused row pass + KeyMult
    with the key ahead of the row pass / L1-prefetched / L1-prefetched one
    digit ahead / staged in shared memory per (row, tile); CK32_TC=0: BConv
    on the CUDA cores (k_bconv) instead of tcgen05; CK32_COL=3/4: the TMA
    column pass k_col / k_col_tma; CK32_KM=12: k_row_keymult8b (4 batch
    items per CTA sharing the row's key slice and twiddles); CK32_TAIL_GATHER=1:
    the one-coefficient-per-thread gather HRot tail -- NTT round trip, HMult (merged and lazy) and HRot equal the
    oracle."""
    import subprocess
    import sys
    from pathlib import Path

    code = f'''
import sys, numpy as np, torch
sys.path[:0] = {[str(Path(__file__).resolve().parent.parent), str(Path(__file__).resolve().parent.parent / "oracle")]!r}
from fractions import Fraction
from paper_2407_13055_b200 import ckks
from pyoracle import Oracle, Rng
n, l, a, db, level = 1 << 16, 24, 8, 55, {level}
O = Oracle(n, l, a, db)
dev = lambda v: torch.from_numpy(np.ascontiguousarray(v.astype(np.int32))).cuda()
C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db))
g = O.gidx(level, 3)
x = O.random_rows(Rng(level), g)
p = ckks.Polynomial(dev(x), level, 3, ckks.COEFFICIENT, False)
ckks.ntt_forward(C, p)
f = O.ntt_fwd(x, g)
assert np.array_equal(p.data.cpu().numpy().astype(np.uint32), O.canonical(f, g))
ckks.intt_inverse(C, p)
assert np.array_equal(p.data.cpu().numpy().astype(np.uint32), x.astype(np.uint32))
C.close()
xb, xa, yb, ya, evk = O.synthetic(level, 4242 + level)
for lazy in (False, True):
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db, lazy_rescale=lazy))
    xc = ckks.Ciphertext(dev(np.stack([xb, xa])), Fraction(1 << db), level)
    yc = ckks.Ciphertext(dev(np.stack([yb, ya])), Fraction(1 << db), level)
    got = ckks.hmult(C, xc, yc, ckks.EvaluationKey(dev(evk))).data.cpu().numpy().astype(np.uint32)
    ob, oa = O.hmult(level, xb, xa, yb, ya, evk, lazy=lazy)
    lo = level if lazy else level - 2
    assert np.array_equal(got, np.stack([O.canonical(ob, O.gidx(lo)), O.canonical(oa, O.gidx(lo))])), lazy
    if not lazy:
        got = ckks.hrot(C, xc, 5, ckks.EvaluationKey(dev(evk), ckks.ROTATION, 5)).data.cpu().numpy().astype(np.uint32)
        ob, oa = O.hrot(level, xb, xa, 5, evk)
        assert np.array_equal(got, np.stack([O.canonical(ob, O.gidx(level)), O.canonical(oa, O.gidx(level))]))
    C.close()
print("variant ok")
'''
    k, v = variant.split("=")
    env = dict(__import__("os").environ, **{k: v})
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("level,p_rows", [(8, 0), (5, 3)])
def test_ew_raw_representation_matches_reference_formulas(level, p_rows):
    """ck_ew_binary ops 4 / 5 / 6 and ck_ew_mul_const_raw: the reference's
    raw signed lazy int32 arithmetic (poly.cpp:121-180: narrow() after the
    add / sub, signed Montgomery mont_mul, modarith.hpp:20-36) bit for bit on
    values in (-q, q), restated here in numpy."""
    import ctypes
    from paper_2407_13055_b200 import _native as nat

    n, l, a = 1024, 8, 3
    C = ctx_for(n, l, a, 55)
    rows = list(range(level)) + [l + j for j in range(p_rows)]
    q = np.array([int(C.primes[g]) for g in rows], np.int64)[:, None]
    rng = np.random.default_rng(level * 7 + p_rows)
    x = rng.integers(-q + 1, q, (len(rows), n))
    y = rng.integers(-q + 1, q, (len(rows), n))
    qinv = np.array([pow(int(v), -1, 1 << 32) for v in q[:, 0]], np.int64)[:, None]

    def narrow(v):
        return np.where(v >= q, v - q, np.where(v <= -q, v + q, v))

    def mred(v):  # modarith.hpp:20-29 on int64 numpy values
        hi = v >> 32
        t = ((v & 0xFFFFFFFF) * qinv) & 0xFFFFFFFF
        t = np.where(t >= 1 << 31, t - (1 << 32), t)
        return hi - ((t * q) >> 32)

    dx = torch.from_numpy(x.astype(np.int32)).cuda()
    dy = torch.from_numpy(y.astype(np.int32)).cuda()
    for op, want in ((4, narrow(x + y)), (5, narrow(x - y)), (6, mred(x * y))):
        out = torch.empty_like(dx)
        nat.call("ck_ew_binary", C.handle, op, dx.data_ptr(), dy.data_ptr(), out.data_ptr(), level, p_rows, C.stream())
        np.testing.assert_array_equal(out.cpu().numpy().astype(np.int64), want, err_msg=f"op {op}")
    consts = rng.integers(0, 1 << 31, len(rows))
    out = torch.empty_like(dx)
    nat.call("ck_ew_mul_const_raw", C.handle, dx.data_ptr(), nat.u32_array(consts), out.data_ptr(), level, p_rows,
             C.stream())
    c32 = np.where(consts >= 1 << 31, consts - (1 << 32), consts)[:, None]
    np.testing.assert_array_equal(out.cpu().numpy().astype(np.int64), mred(x * c32))


@pytest.mark.parametrize("n,level", [(64, 3), (1024, 8)])
def test_ntt_raw_representation_matches_reference_serial(n, level):
    """ck_ntt_forward_raw / ck_intt_inverse_raw: the reference's serial NTT in
    its raw signed lazy representation (ntt.cpp:15-96, forward_row_serial /
    inverse_row_serial), restated here in numpy stage by stage with the
    reference's table (ntt.cpp:100-135) -- equal int32 for int32, and the
    inverse with an epilogue constant canonical."""
    from paper_2407_13055_b200 import _native as nat

    C = ctx_for(n, 8, 3, 55)
    logn = n.bit_length() - 1
    g = list(range(level))
    rng = np.random.default_rng(n + level)

    def brev(i):
        return int(format(i, f"0{logn}b")[::-1], 2)

    def mred(v, q, m):  # modarith.hpp:20-29, int64 numpy
        hi = v >> 32
        t = ((v & 0xFFFFFFFF) * m) & 0xFFFFFFFF
        t = np.where(t >= 1 << 31, t - (1 << 32), t)
        return hi - ((t * q) >> 32)

    def narrow(v, b):
        return np.where(v >= b, v - b, np.where(v <= -b, v + b, v))

    def find_root_2n(q):  # modarith.cpp:30-40: first g >= 2 whose cofactor power has order 2n
        cof = (q - 1) // (2 * n)
        for gg in range(2, q):
            cand = pow(gg, cof, q)
            if pow(cand, n, q) == q - 1:
                return cand

    x0 = np.stack([rng.integers(-int(C.primes[i]) + 1, int(C.primes[i]), n) for i in g]).astype(np.int64)
    want_f, want_i = [], []
    epi = [int(rng.integers(1, int(C.primes[i]))) for i in g]
    for r, gi in enumerate(g):
        q = int(C.primes[gi]); m = pow(q, -1, 1 << 32); R = (1 << 32) % q; r2 = R * R % q
        psi = find_root_2n(q)
        pw = [pow(psi, k, q) for k in range(n)]
        pwi = [pow(psi, -k, q) for k in range(n)]
        fwd = [0] + [pw[brev(i)] * R % q for i in range(1, n)]
        inv = [0] + [pwi[brev(i)] * R % q for i in range(1, n)]
        fwd1_r2 = pw[n // 2] * R % q * R % q
        ninv = pow(n, -1, q)
        exit_x, exit_y = ninv, pwi[n // 2] * ninv % q
        a = x0[r].copy()
        for s in range(logn):  # fwd_stages, one stage at a time (forward_row_serial)
            mm, t = 1 << s, n >> (s + 1)
            for gg in range(mm):
                w = fwd1_r2 if s == 0 else fwd[mm + gg]
                xs = a[2 * gg * t:2 * gg * t + t].copy()
                ys = mred(a[2 * gg * t + t:2 * gg * t + 2 * t] * w, q, m)
                if s == 0:
                    xs = mred(xs * r2, q, m)
                u, v = narrow(xs + ys, 2 * q), narrow(xs - ys, 2 * q)
                if s == logn - 1:
                    u, v = narrow(u, q), narrow(v, q)
                a[2 * gg * t:2 * gg * t + t], a[2 * gg * t + t:2 * gg * t + 2 * t] = u, v
        want_f.append(a.copy())
        for s in range(logn):  # inv_stages (inverse_row_serial) with the epilogue
            mm, t = n >> (1 + s), 1 << s
            for gg in range(mm):
                xs = a[2 * gg * t:2 * gg * t + t].copy()
                ys = a[2 * gg * t + t:2 * gg * t + 2 * t].copy()
                u, v2 = xs + ys, xs - ys
                if mm == 1:
                    a0, a1 = mred(u * exit_x, q, m), mred(v2 * exit_y, q, m)
                    a0, a1 = mred(a0 * epi[r], q, m), mred(a1 * epi[r], q, m)
                    a0, a1 = np.where(a0 < 0, a0 + q, a0), np.where(a1 < 0, a1 + q, a1)
                    a[2 * gg * t:2 * gg * t + t], a[2 * gg * t + t:2 * gg * t + 2 * t] = a0, a1
                else:
                    a[2 * gg * t:2 * gg * t + t] = narrow(u, 2 * q)
                    a[2 * gg * t + t:2 * gg * t + 2 * t] = mred(v2 * inv[mm + gg], q, m)
        want_i.append(a.copy())
    d = torch.from_numpy(x0.astype(np.int32)).cuda()
    garr = nat.u32_array(g)
    nat.call("ck_ntt_forward_raw", C.handle, d.data_ptr(), level, garr, C.stream())
    np.testing.assert_array_equal(d.cpu().numpy().astype(np.int64), np.stack(want_f))
    nat.call("ck_intt_inverse_raw", C.handle, d.data_ptr(), level, garr, nat.u32_array(epi), C.stream())
    np.testing.assert_array_equal(d.cpu().numpy().astype(np.int64), np.stack(want_i))


def test_raw_entry_points_argument_errors():
    """The raw-representation entry points validate like the rest of the ABI:
    a prime index past the basis, a null prime list with rows, and an
    element-wise op code outside 0-2 / 4-6 raise ValueError."""
    from paper_2407_13055_b200 import _native as nat

    C = ctx_for(1024, 8, 3, 55)
    d = torch.zeros((2, 1024), dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        nat.call("ck_ntt_forward_raw", C.handle, d.data_ptr(), 2, nat.u32_array([0, 99]), C.stream())
    with pytest.raises(ValueError):
        nat.call("ck_intt_inverse_raw", C.handle, d.data_ptr(), 2, None, None, C.stream())
    for op in (3, 7, -1):
        with pytest.raises(ValueError):
            nat.call("ck_ew_binary", C.handle, op, d.data_ptr(), d.data_ptr(), d.data_ptr(), 2, 0, C.stream())
