"""CPU suite: pins the C restatement (oracle/ck32_oracle.c) against the
reference's own golden fixtures and full-size hashes, checks the wire formats
round-trip byte-exactly, and (when oracle/_ref exists) runs the reference's
own unit tests against the shims.  No GPU needed."""
from __future__ import annotations

import subprocess
from fractions import Fraction

import numpy as np
import pytest

from golden_util import FULL, SMALL_DIRS, Fixture, full_cases, sha
from paper_2407_13055_b200 import wire
from pyoracle import REF_DIR, Oracle, Reference, Rng, generate_basis

SMALL = [pytest.param(d, id=d.name) for d in SMALL_DIRS]


def canon(O, rows, level, p_rows=0):
    return O.canonical(rows, O.gidx(level, p_rows))


def test_mt19937_64_matches_std():
    # first output of std::mt19937_64 default seed 5489 is 14514284786278117030 (C++ standard [rand.predef])
    assert Rng(5489).next() == 14514284786278117030


@pytest.mark.parametrize("cfg", [(65536, 24, 8, 55), (131072, 24, 8, 55), (1 << 16, 54, 14, 48), (256, 6, 2, 48)])
def test_basis_matches_golden_or_reference(cfg):
    n, l, a, db = cfg
    got = generate_basis(n, l, a, db)
    assert len(got) == l + a
    assert all(int(p) % (2 * n) == 1 and int(p) < (1 << 29) for p in got)
    if Reference.available:
        np.testing.assert_array_equal(got, Reference().basis(n, l, a, db))


@pytest.mark.parametrize("d", SMALL)
def test_oracle_basis_equals_fixture(d):
    fx = Fixture(d)
    np.testing.assert_array_equal(generate_basis(fx.n, fx.l, fx.alpha, fx.db), fx.basis.primes)


@pytest.mark.parametrize("d", SMALL)
def test_wire_roundtrip_byte_exact(d):
    for f in sorted(d.glob("*.bin")):
        b = f.read_bytes()
        magic = int.from_bytes(b[:4], "little")
        if magic == wire.CT_MAGIC:
            assert wire.write_ciphertext(wire.read_ciphertext(b)) == b
        elif magic == wire.EVK_MAGIC:
            assert wire.write_evk(wire.read_evk(b)) == b
        elif magic == wire.POLY_MAGIC:
            assert wire.write_poly(wire.read_poly(b)[0]) == b
        elif magic == wire.BASIS_MAGIC:
            bb = wire.read_basis(b)
            assert wire.write_basis(bb) == b
        else:
            raise AssertionError(f"unknown blob {f}")


def test_wire_rejects_corruption():
    d = SMALL_DIRS[0]
    b = bytearray((d / "basis.bin").read_bytes())
    b[0] ^= 0xFF
    with pytest.raises(RuntimeError):
        wire.read_basis(bytes(b))
    with pytest.raises(ValueError):
        wire.read_ciphertext(b"\x00" * 16)
    p = (d / "sk.bin").read_bytes()
    with pytest.raises(RuntimeError):
        wire.read_poly(p[:-8])


@pytest.mark.parametrize("d", SMALL)
def test_basis_hash_matches_poly_headers(d):
    fx = Fixture(d)
    assert fx.poly("sk").basis_hash == fx.basis.hash


@pytest.mark.parametrize("d", SMALL)
def test_oracle_mechanisms_equal_reference_fixtures(d):
    fx = Fixture(d)
    O = Oracle(fx.n, fx.l, fx.alpha, fx.db)
    np.testing.assert_array_equal(O.primes, fx.basis.primes)
    l, a = fx.l, fx.alpha
    u, v = fx.ct("ct_u"), fx.ct("ct_v")
    ub, ua, vb, va = (x.rows.astype(np.int32) for x in (u.b, u.a, v.b, v.a))
    relin = fx.evk("evk_relin").stacked().astype(np.int32)
    rot1 = fx.evk("evk_rot1").stacked().astype(np.int32)
    rot3 = fx.evk("evk_rot3").stacked().astype(np.int32)

    def eq(name, b_rows, a_rows, level):
        ref = fx.ct(name)
        assert ref.level == level
        np.testing.assert_array_equal(canon(O, b_rows, level), ref.b.rows, err_msg=name)
        np.testing.assert_array_equal(canon(O, a_rows, level), ref.a.rows, err_msg=name)

    eq("out_hmult", *O.hmult(l, ub, ua, vb, va, relin), l - 2)
    eq("out_hmult_lazy", *O.hmult(l, ub, ua, vb, va, relin, lazy=True), l)
    eq("out_hrot1", *O.hrot(l, ub, ua, 1, rot1), l)
    eq("out_hrot3", *O.hrot(l, ub, ua, 3, rot3), l)
    eq("out_rescale", *O.rescale(l, ub, ua), l - 2)
    eq("out_hadd", _ew_add(O, l, ub, vb), _ew_add(O, l, ua, va), l)
    pt = fx.poly("pt_v").rows.astype(np.int32)
    eq("out_pmult", _ew_mul(O, l, ub, pt), _ew_mul(O, l, ua, pt), l)
    eq("out_padd", _ew_add(O, l, ub, pt), ua, l)

    h = O.mod_up(l, ua)
    for k in range(O.digits(l)):
        np.testing.assert_array_equal(canon(O, h[k], l, a), fx.poly(f"out_modup_d{k}").rows)
    v0, v1 = O.key_mult(l, h, relin)
    np.testing.assert_array_equal(canon(O, v0, l, a), fx.poly("out_keymult_v0").rows)
    np.testing.assert_array_equal(canon(O, v1, l, a), fx.poly("out_keymult_v1").rows)
    np.testing.assert_array_equal(canon(O, O.mod_down(l, v0), l), fx.poly("out_moddown_v0").rows)
    c0, c1 = O.key_switch(l, ua, relin)
    np.testing.assert_array_equal(canon(O, c0, l), fx.poly("out_keyswitch_c0").rows)
    np.testing.assert_array_equal(canon(O, c1, l), fx.poly("out_keyswitch_c1").rows)

    pts = [fx.poly(f"pt_acc{i}").rows.astype(np.int32) for i in range(3)]
    eq("out_hoisted_acc", *O.hoisted_accumulate(l, ub, ua, [0, 1, 3], pts, [None, rot1, rot3]), l)
    eq("out_hoisted_r1", *O.hrot(l, ub, ua, 1, rot1), l)

    coeff = fx.poly("in_ntt_coeff")
    g = O.gidx(l, a)
    np.testing.assert_array_equal(canon(O, O.ntt_fwd(coeff.rows.astype(np.int32), g), l, a),
                                  fx.poly("out_ntt_coeff").rows)
    np.testing.assert_array_equal(canon(O, O.intt(ub, O.gidx(l)), l), fx.poly("out_intt_ctub").rows)


def _ew_add(O, l, x, y):
    o = np.zeros_like(x)
    O.lib.cko_ew_add(O._c, l, np.ascontiguousarray(x), np.ascontiguousarray(y), o)
    return o


def _ew_mul(O, l, x, y):
    o = np.zeros_like(x)
    O.lib.cko_ew_mul(O._c, l, np.ascontiguousarray(x), np.ascontiguousarray(y), o)
    return o


@pytest.mark.parametrize("d", SMALL)
def test_fixture_ledger(d):
    # scale ledger of the reference outputs (ckks.cpp:797-851)
    fx = Fixture(d)
    u, v = fx.ct("ct_u"), fx.ct("ct_v")
    q = [int(x) for x in fx.basis.primes]
    qq = q[fx.l - 2] * q[fx.l - 1]
    assert u.scale == Fraction(1 << fx.db)
    assert fx.ct("out_hmult").scale == u.scale * v.scale / qq
    assert fx.ct("out_rescale").scale == u.scale / qq
    lazy = fx.ct("out_hmult_lazy")
    assert lazy.pending_rescale and lazy.scale == u.scale * v.scale


FULL_CPU = [c for c in full_cases() if c[0] == "n65536_l24_a8_d55" and c[2:5] in
            [("hmult", 24, 0), ("hrot", 24, 1), ("ntt", 24, 0)]]


@pytest.mark.parametrize("case", FULL_CPU, ids=[f"{c[2]}@{c[3]}@{c[4]}" for c in FULL_CPU])
def test_oracle_full_size_hash(case):
    name, cfg, op, level, rot, h = case
    O = Oracle(cfg["n"], cfg["l"], cfg["alpha"], cfg["delta_bits"])
    xb, xa, yb, ya, evk = O.synthetic(level, FULL["seed"])
    if op == "hmult":
        ob, oa = O.hmult(level, xb, xa, yb, ya, evk)
        got = np.concatenate([canon(O, ob, level - 2), canon(O, oa, level - 2)])
    elif op == "hrot":
        ob, oa = O.hrot(level, xb, xa, rot, evk)
        got = np.concatenate([canon(O, ob, level), canon(O, oa, level)])
    else:
        got = canon(O, O.ntt_fwd(xb, O.gidx(level)), level)
    assert sha(got) == h


@pytest.mark.skipif(not (REF_DIR / "ref_unit_tests").exists(), reason="reference not built here")
def test_reference_unit_suite_passes_against_shims():
    r = subprocess.run([str(REF_DIR / "ref_unit_tests")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "test cases failed: 0" in r.stdout


@pytest.mark.parametrize("n", [16, 256])
def test_oracle_automorphism_restatement(n):
    """cko_automorphism: the evaluation-domain gather for a rotation's Galois
    element equals the rotation map (automorphism.cpp:38-69), conjugation is an
    involution, and the coefficient-domain variant commutes with the NTT
    (the reference's own property, test_automorphism.cpp:71-96)."""
    from pyoracle import Oracle, Rng

    O = Oracle(n, 4, 2, 48)
    g = O.gidx(4, 2)
    x = O.random_rows(Rng(n), g)
    for r in (1, -3, 5):
        gal = pow(5, (-r) % (n // 2), 2 * n)
        np.testing.assert_array_equal(O.automorphism(x, gal, False), x[:, O.rotation_src_map(r)])
        lhs = O.ntt_fwd(O.automorphism(x, gal, True), g)
        rhs = O.automorphism(O.ntt_fwd(x, g), gal, False)
        np.testing.assert_array_equal(O.canonical(lhs, g), O.canonical(rhs, g))
    conj = 2 * n - 1
    for coeff in (False, True):
        twice = O.automorphism(O.automorphism(x, conj, coeff), conj, coeff)
        np.testing.assert_array_equal(O.canonical(twice, g), O.canonical(x, g))


def test_oracle_elementwise_restatement():
    """cko_ew_rows over P-extended rows: add/sub round trip, mul by the
    Montgomery one R mod q is the identity, mul_const by R is the identity."""
    from pyoracle import Oracle, Rng

    O = Oracle(64, 4, 2, 48)
    g = O.gidx(3, 2)
    x, y = O.random_rows(Rng(1), g), O.random_rows(Rng(2), g)
    s = O.ew(0, x, y, g)
    np.testing.assert_array_equal(O.canonical(O.ew(1, s, y, g), g), O.canonical(x, g))
    R = [(1 << 32) % int(q) for q in O.primes[g]]
    one = np.repeat(np.array(R, np.int64)[:, None], 64, 1)
    np.testing.assert_array_equal(O.canonical(O.ew(2, x, one, g), g), O.canonical(x, g))
    np.testing.assert_array_equal(O.canonical(O.ew(3, x, None, g, R), g), O.canonical(x, g))
