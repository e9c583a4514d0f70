"""Encrypt / decrypt element-wise parts on the GPU (ckks.cpp:497-553, SURVEY
§8(a) row a23) and an end-to-end precision check through the GPU evaluator:
the reference's own keys and ciphertexts (golden fixtures), decrypted on the
GPU, decoded on the GPU, compared with the slots the reference encoded."""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

from golden_util import SMALL_DIRS, Fixture

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2407_13055_b200 import ckks  # noqa: E402

_CTX = {}


def ctx_of(F):
    key = (F.n, F.l, F.alpha, F.db)
    if key not in _CTX:
        _CTX[key] = ckks.CkksContext(ckks.CkksParams(n=F.n, l=F.l, alpha=F.alpha, delta_bits=F.db))
    return _CTX[key]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).astype(np.int64).astype(np.int32))).cuda()


def slots(F, name):
    raw = np.frombuffer((F.dir / f"{name}.f64").read_bytes(), dtype=np.float64)
    return raw[0::2] + 1j * raw[1::2]


def gpu_ct(F, name):
    c = F.ct(name)
    return ckks.Ciphertext(dev(F.ct_rows(c)), c.scale, c.level)


@pytest.mark.parametrize("d", SMALL_DIRS, ids=lambda p: p.name)
def test_decrypt_equals_reference(d):
    F = Fixture(d)
    C = ctx_of(F)
    s = dev(F.poly("sk").rows)
    got = ckks.decrypt(C, gpu_ct(F, "ct_u"), s).poly.data.cpu().numpy().astype(np.uint32)
    np.testing.assert_array_equal(got, F.poly("out_decrypt_u").rows.astype(np.uint32))


@pytest.mark.parametrize("d", SMALL_DIRS, ids=lambda p: p.name)
def test_hmult_end_to_end_precision(d):
    """reference keys + ciphertexts -> GPU HMult -> GPU decrypt (== the
    reference's decrypt of its own HMult) -> GPU decode ~ u * v."""
    F = Fixture(d)
    C = ctx_of(F)
    s = dev(F.poly("sk").rows)
    ev = F.evk("evk_relin")
    K = ckks.EvaluationKey(dev(np.stack([np.stack([b.rows, a.rows]) for b, a in ev.digits])))
    m = ckks.hmult(C, gpu_ct(F, "ct_u"), gpu_ct(F, "ct_v"), K)
    pt = ckks.decrypt(C, m, s)
    np.testing.assert_array_equal(pt.poly.data.cpu().numpy().astype(np.uint32),
                                  F.poly("out_decrypt_hmult").rows.astype(np.uint32))
    if pt.level >= 1:
        got = ckks.decode(C, pt)
        want = slots(F, "slots_u") * slots(F, "slots_v")
        assert np.abs(got - want).max() < 2.0 ** -12  # delta = 2^48 at N <= 1024


@pytest.mark.parametrize("d", SMALL_DIRS, ids=lambda p: p.name)
def test_encrypt_sk_pk_round_trip(d):
    F = Fixture(d)
    C = ctx_of(F)
    s = dev(F.poly("sk").rows)
    rng = np.random.default_rng(7)
    z = slots(F, "slots_u")
    l = F.l
    pt = ckks.encode(C, z, Fraction(1 << F.db), l)
    a = ckks.uniform_eval(C, l, rng)
    e = ckks.coeffs_to_eval(C, ckks.sample_gaussian(F.n, 3.2, rng), l)
    ct = ckks.encrypt_sk(C, pt, s, a, e)
    m = ckks.decrypt(C, ct, s)
    # exact identity: decrypt(encrypt(m; a, e)) = m + e (evaluation domain)
    want = ckks.ew_add(C, ckks.Polynomial(pt.poly.data, l), ckks.Polynomial(e.data, l))
    np.testing.assert_array_equal(m.poly.data.cpu().numpy(), want.data.cpu().numpy())
    assert np.abs(ckks.decode(C, m) - z).max() < 2.0 ** -30
    # public key = secret-key encryption of zero at the top level; encrypt with it
    zero = ckks.encode(C, [], Fraction(1 << F.db), l)
    pk = ckks.encrypt_sk(C, zero, s, ckks.uniform_eval(C, l, rng),
                         ckks.coeffs_to_eval(C, ckks.sample_gaussian(F.n, 3.2, rng), l))
    v = ckks.coeffs_to_eval(C, ckks.sample_ternary(F.n, min(64, F.n // 4), rng), l)
    e0 = ckks.coeffs_to_eval(C, ckks.sample_gaussian(F.n, 3.2, rng), l)
    e1 = ckks.coeffs_to_eval(C, ckks.sample_gaussian(F.n, 3.2, rng), l)
    ct2 = ckks.encrypt_pk(C, pt, pk, v, e0, e1)
    assert np.abs(ckks.decode(C, ckks.decrypt(C, ct2, s)) - z).max() < 2.0 ** -25
