"""Key generation on the GPU (keygen / pubkey_gen / evk_gen, ckks.cpp:399-477;
host-sampled randomness) and a fully GPU-side encrypted round trip:
encode -> public-key encrypt -> HMult+relin / HRot -> decrypt -> decode,
compared with the plaintext slot arithmetic within CKKS precision."""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2407_13055_b200 import ckks  # noqa: E402


def unit(count, rng):
    r = rng.uniform(-1.0, 1.0, (count, 2))
    return r[:, 0] + 1j * r[:, 1]


@pytest.mark.parametrize("n,l,a,db", [(1024, 8, 3, 48), (8192, 12, 4, 48)])
def test_gpu_keys_encrypted_round_trip(n, l, a, db):
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db))
    rng = np.random.default_rng(2024 + n)
    s = ckks.keygen(C, rng)
    assert s.shape == (l + a, n)
    pk = ckks.pubkey_gen(C, s, rng)
    relin = ckks.evk_gen(C, s, ckks.RELIN, 0, rng)
    rot = ckks.evk_gen(C, s, ckks.ROTATION, 3, rng)
    delta = Fraction(1 << db)

    def enc(z):
        pt = ckks.encode(C, z, delta, l)
        v = ckks.coeffs_to_eval(C, ckks.sample_ternary(n, min(64, n // 4), rng), l)
        e0 = ckks.coeffs_to_eval(C, ckks.sample_gaussian(n, 3.2, rng), l)
        e1 = ckks.coeffs_to_eval(C, ckks.sample_gaussian(n, 3.2, rng), l)
        return ckks.encrypt_pk(C, pt, pk, v, e0, e1)

    def dec(ct):
        return ckks.decode(C, ckks.decrypt(C, ct, s))

    z1, z2 = unit(n // 2, rng), unit(n // 2, rng)
    c1, c2 = enc(z1), enc(z2)
    assert np.abs(dec(c1) - z1).max() < 2.0 ** -20
    prod = ckks.hmult(C, c1, c2, relin)
    assert np.abs(dec(prod) - z1 * z2).max() < 2.0 ** -12
    r = ckks.hrot(C, c1, 3, rot)
    assert np.abs(dec(r) - np.roll(z1, -3)).max() < 2.0 ** -12
    # depth: a second multiplication on the product
    prod2 = ckks.hmult(C, prod, ckks.hmult(C, c2, c2, relin), relin)
    assert np.abs(dec(prod2) - z1 * z2 ** 3).max() < 2.0 ** -8
    C.close()


from golden_util import SMALL_DIRS, SMALL_SEEDS, Fixture, parse_small_name, ref_unit_slots  # noqa: E402


@pytest.mark.parametrize("d", SMALL_DIRS, ids=lambda p: p.name)
def test_reference_rng_reproduces_reference_keys_and_ciphertexts(d):
    """With the reference's randomness (ckks.RefRng = std::mt19937_64(seed)
    consumed as ckks.cpp does) the GPU keygen / evk_gen / encode / encrypt
    reproduce the reference's own fixtures bit for bit: sk.s, the relin and
    rotation keys, and both secret-key ciphertexts (ref_driver.cpp
    ref_gen_fixtures order)."""
    F = Fixture(d)
    n, l, a = parse_small_name(d)
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=F.db))
    rng = ckks.RefRng(SMALL_SEEDS[(n, l, a)])
    s = ckks.keygen(C, rng)
    np.testing.assert_array_equal(s.cpu().numpy().astype(np.uint32), F.poly("sk").rows)
    for name, kind, r in (("evk_relin", ckks.RELIN, 0), ("evk_rot1", ckks.ROTATION, 1), ("evk_rot3", ckks.ROTATION, 3)):
        k = ckks.evk_gen(C, s, kind, r, rng)
        np.testing.assert_array_equal(k.data.cpu().numpy().astype(np.uint32), F.evk(name).stacked(), err_msg=name)
    u = ref_unit_slots(rng.draws(n))
    v = ref_unit_slots(rng.draws(n))
    for name, z in (("ct_u", u), ("ct_v", v)):
        ct = ckks.encrypt(C, ckks.encode(C, z, C.default_scale(), l), s, rng)
        want = F.ct(name)
        np.testing.assert_array_equal(ct.data.cpu().numpy().astype(np.uint32), Fixture.ct_rows(want), err_msg=name)
        assert ct.scale == want.scale and ct.level == want.level
    C.close()


def test_reference_rng_public_key_encrypt_decrypts():
    """pubkey_gen + public-key encrypt with the reference's stream (v, e0, e1
    order of ckks.cpp:523-526) decrypt to the message."""
    n, l, a, db = 1024, 8, 3, 48
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db))
    rng = ckks.RefRng(99)
    s = ckks.keygen(C, rng)
    pk = ckks.pubkey_gen(C, s, rng)
    z = ref_unit_slots(rng.draws(n))
    ct = ckks.encrypt(C, ckks.encode(C, z, C.default_scale(), l), pk, rng)
    back = ckks.decode(C, ckks.decrypt(C, ct, s))
    assert np.abs(back - z).max() < 2.0 ** -20
    C.close()


def test_baby_step_linear_transform_16x16_like_reference():
    """test_ckks.cpp:468-503 on the GPU, with the reference's own inputs: the
    same toy parameters (n=32, l=4, alpha=2, delta 2^48), the same
    std::mt19937_64(211) stream consumed in the same order (keygen, x, the
    16x16 matrix, encrypt, then per rotation evk_gen), the diagonals encoded
    P-extended, one hoisted_rotate_accumulate; decrypted M x within 1e-4."""
    n, l, a = 32, 4, 2
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=48))
    rng = ckks.RefRng(211)
    s = ckks.keygen(C, rng)
    slots = n // 2
    x = ref_unit_slots(rng.draws(2 * slots))
    m = [ref_unit_slots(rng.draws(2 * slots)) for _ in range(slots)]
    ct = ckks.encrypt(C, ckks.encode(C, x, C.default_scale(), l), s, rng)
    keys, diags = [], []
    for r in range(slots):
        keys.append(ckks.evk_gen(C, s, ckks.ROTATION, r, rng) if r else None)
        diag = np.array([m[t][(t + r) % slots] for t in range(slots)])
        diags.append(ckks.encode(C, diag, C.default_scale(), l, p_extend=True))
    y_ct = ckks.hoisted_rotate_accumulate(C, ct, list(range(slots)), diags, keys)
    y = ckks.decode(C, ckks.decrypt(C, y_ct, s))
    want = np.array([sum(m[t][j] * x[j] for j in range(slots)) for t in range(slots)])
    assert np.abs(y - want).max() < 1e-4
    C.close()


def test_acceptance_c7_noise_bound_default_params():
    """Acceptance criterion C7 (acceptance_main.cpp:303-350) on the GPU with
    the reference's own inputs: default parameters (N=2^16, L=54, alpha=14,
    delta 2^48), keys from mt19937_64(42) (keygen, relin, rot 1), 100 message
    seeds mt19937_64(1000 + seed) (u, v, encrypt u, encrypt v); hadd,
    pmult + rescale, hmult, hrot(1) all decrypt within 2^-20."""
    C = ckks.CkksContext(ckks.CkksParams())
    key_rng = ckks.RefRng(42)
    s = ckks.keygen(C, key_rng)
    relin = ckks.evk_gen(C, s, ckks.RELIN, 0, key_rng)
    rot1 = ckks.evk_gen(C, s, ckks.ROTATION, 1, key_rng)
    slots, l, D = C.n // 2, C.params.l, C.default_scale()
    dec = lambda ct: ckks.decode(C, ckks.decrypt(C, ct, s))
    err = {"hadd": 0.0, "pmult": 0.0, "hmult": 0.0, "hrot": 0.0}
    for seed in range(100):
        rng = ckks.RefRng(1000 + seed)
        u = ref_unit_slots(rng.draws(2 * slots))
        v = ref_unit_slots(rng.draws(2 * slots))
        pt_u, pt_v = ckks.encode(C, u, D, l), ckks.encode(C, v, D, l)
        cu = ckks.encrypt(C, pt_u, s, rng)
        cv = ckks.encrypt(C, pt_v, s, rng)
        err["hadd"] = max(err["hadd"], np.abs(dec(ckks.hadd(C, cu, cv)) - (u + v)).max())
        err["pmult"] = max(err["pmult"], np.abs(dec(ckks.rescale(C, ckks.pmult(C, cu, pt_v))) - u * v).max())
        err["hmult"] = max(err["hmult"], np.abs(dec(ckks.hmult(C, cu, cv, relin)) - u * v).max())
        err["hrot"] = max(err["hrot"], np.abs(dec(ckks.hrot(C, cu, 1, rot1)) - np.roll(u, -1)).max())
    assert max(err.values()) <= 2.0 ** -20, err
    C.close()


def test_acceptance_c8_hoisting_counters():
    """Acceptance C8 (acceptance_main.cpp:354-408) on the GPU with the
    reference's inputs (n=2^10, l=8, alpha=2, h=64, mt19937_64(29)): 8
    separate HRots cost 8 ModUps, hoisted_rotations 1, and
    hoisted_rotate_accumulate 1 ModUp + 1 ModDown."""
    C = ckks.CkksContext(ckks.CkksParams(n=1024, l=8, alpha=2, delta_bits=48, hamming=64))
    rng = ckks.RefRng(29)
    s = ckks.keygen(C, rng)
    rots = list(range(1, 9))
    keys = [ckks.evk_gen(C, s, ckks.ROTATION, r, rng) for r in rots]
    u = ref_unit_slots(rng.draws(C.n))
    ct = ckks.encrypt(C, ckks.encode(C, u, C.default_scale(), 8), s, rng)
    C.reset_counters()
    outs = [ckks.hrot(C, ct, r, k) for r, k in zip(rots, keys)]
    unhoisted = C.counters()["modup"]
    C.reset_counters()
    hoisted = ckks.hoisted_rotations(C, ct, rots, keys)
    assert C.counters()["modup"] == 1 and unhoisted == 8
    for a, b in zip(outs, hoisted):  # singleton-hoist == hrot, bit-exact (test_ckks.cpp:382-466)
        assert torch.equal(a.data, b.data)
    pts = [ckks.encode(C, np.full(C.n // 2, 0.125 * (i + 1)), C.default_scale(), 8, p_extend=True)
           for i in range(len(rots))]
    C.reset_counters()
    acc = ckks.hoisted_rotate_accumulate(C, ct, rots, pts, keys)
    c = C.counters()
    assert (c["modup"], c["moddown"]) == (1, 1)
    want = sum(0.125 * (i + 1) * np.roll(u, -r) for i, r in enumerate(rots))
    back = ckks.decode(C, ckks.decrypt(C, acc, s))
    assert np.abs(back - want).max() < 1e-6
    C.close()


def test_acceptance_c9_merged_vs_lazy_hmult():
    """Acceptance C9 (acceptance_main.cpp:413-478) on the GPU with the
    reference's inputs: n=2^12, l=12, alpha=3, h=128, keys mt19937_64(7) in
    a merged and a lazy-rescale context, 50 message seeds (500 + seed); the
    lazy path defers the rescale, the flushed ledgers are identical, the two
    decryptions agree within their combined noise and the noise bounds stay
    within 4x of each other."""
    base = dict(n=4096, l=12, alpha=3, delta_bits=48, hamming=128)
    Cm = ckks.CkksContext(ckks.CkksParams(**base))
    Cu = ckks.CkksContext(ckks.CkksParams(**base, lazy_rescale=True))
    kr_m, kr_u = ckks.RefRng(7), ckks.RefRng(7)
    sk_m, sk_u = ckks.keygen(Cm, kr_m), ckks.keygen(Cu, kr_u)
    relin_m = ckks.evk_gen(Cm, sk_m, ckks.RELIN, 0, kr_m)
    relin_u = ckks.evk_gen(Cu, sk_u, ckks.RELIN, 0, kr_u)
    slots = Cm.n // 2
    bound_m = bound_u = 0.0
    for seed in range(50):
        rng_m, rng_u = ckks.RefRng(500 + seed), ckks.RefRng(500 + seed)
        u = ref_unit_slots(rng_m.draws(2 * slots))
        v = ref_unit_slots(rng_m.draws(2 * slots))
        rng_u.draws(4 * slots)  # the same draws keep both encryption streams aligned

        def enc(C, sk, r, m):
            return ckks.encrypt(C, ckks.encode(C, m, C.default_scale(), 12), sk, r)

        ct_m = ckks.hmult(Cm, enc(Cm, sk_m, rng_m, u), enc(Cm, sk_m, rng_m, v), relin_m)
        ct_l = ckks.hmult(Cu, enc(Cu, sk_u, rng_u, u), enc(Cu, sk_u, rng_u, v), relin_u)
        assert ct_l.pending_rescale
        ct_f = ckks.rescale(Cu, ct_l)
        assert (ct_m.level, ct_m.scale) == (ct_f.level, ct_f.scale)
        dm = ckks.decode(Cm, ckks.decrypt(Cm, ct_m, sk_m))
        du = ckks.decode(Cu, ckks.decrypt(Cu, ct_f, sk_u))
        e_m, e_u = np.abs(dm - u * v).max(), np.abs(du - u * v).max()
        bound_m, bound_u = max(bound_m, e_m), max(bound_u, e_u)
        assert np.abs(dm - du).max() <= e_m + e_u + 1e-12
    assert bound_m <= 4 * bound_u + 1e-12 and bound_u <= 4 * bound_m + 1e-12
    Cm.close()
    Cu.close()


def _crt_centered(rows, primes):
    """CRT-lift canonical coefficient rows [l][n] over `primes`, centred."""
    M = 1
    for q in primes:
        M *= q
    out = []
    for k in range(rows.shape[1]):
        v = 0
        for i, q in enumerate(primes):
            Mi = M // q
            v += int(rows[i, k]) * Mi * pow(Mi, -1, q)
        v %= M
        out.append(v - M if v > M // 2 else v)
    return out, M


def _toy(n=256, l=6, a=2):  # test_ckks.cpp toy_params
    return ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=48, hamming=64))


def test_key_switch_retargets_decryption_like_reference():
    """test_ckks.cpp:155-191 on the GPU with its inputs (mt19937_64(149):
    keygen, relin key, random d): c0 + c1 s - d s^2 has centred coefficients
    within 2^24."""
    C = _toy()
    rng = ckks.RefRng(149)
    s = ckks.keygen(C, rng)
    relin = ckks.evk_gen(C, s, ckks.RELIN, 0, rng)
    l, n = C.params.l, C.n
    primes = [int(q) for q in C.q_primes[:l]]
    d = rng.uniform(primes, n)
    c0, c1 = ckks.key_switch(C, ckks.Polynomial(torch.from_numpy(d.astype(np.int64).astype(np.int32)).cuda(), l),
                             relin)
    S = s[:l].cpu().numpy().astype(np.uint32).astype(object)
    C0 = c0.data.cpu().numpy().astype(np.uint32).astype(object)
    C1 = c1.data.cpu().numpy().astype(np.uint32).astype(object)
    D = d.astype(object)
    e = np.empty((l, n), dtype=np.int64)
    for i, q in enumerate(primes):
        rinv = pow(1 << 32, -1, q)
        got = (C0[i] + C1[i] * S[i] * rinv) % q
        want = (D[i] * S[i] * S[i] * rinv * rinv) % q
        e[i] = ((got - want) % q).astype(np.int64)
    poly = ckks.intt_inverse(C, ckks.Polynomial(torch.from_numpy(e.astype(np.int32)).cuda(), l))
    coeffs, _ = _crt_centered(poly.data.cpu().numpy().astype(np.uint32), primes)
    assert max(abs(x) for x in coeffs) <= 1 << 24
    C.close()


def test_rescale_is_floor_divide_like_reference():
    """test_ckks.cpp:193-237 on the GPU with its inputs (mt19937_64(151):
    keygen, slots, encode, encrypt): after rescale, b's coefficients equal
    floor(v / (q_{l-2} q_{l-1})) - e with e in {0, 1}; level l-2, scale
    divided by q_{l-2} q_{l-1}; a second rescale drops two more primes."""
    C = _toy()
    rng = ckks.RefRng(151)
    s = ckks.keygen(C, rng)
    n, l = C.n, C.params.l
    u = ref_unit_slots(rng.draws(n))
    ct = ckks.encrypt(C, ckks.encode(C, u, C.default_scale(), l), s, rng)
    primes = [int(q) for q in C.q_primes[:l]]
    qq = primes[l - 2] * primes[l - 1]
    before = ckks.intt_inverse(C, ckks.Polynomial(ct.data[0].clone(), l)).data.cpu().numpy().astype(np.uint32)
    rs = ckks.rescale(C, ct)
    assert rs.level == l - 2 and rs.scale == ct.scale / qq
    after = ckks.intt_inverse(C, ckks.Polynomial(rs.data[0].clone(), l - 2)).data.cpu().numpy().astype(np.uint32)
    M_full = 1
    for q in primes:
        M_full *= q
    M_low = M_full // qq
    for k in range(n):
        v = sum(int(before[i, k]) * (M_full // q) * pow(M_full // q, -1, q) for i, q in enumerate(primes)) % M_full
        got = sum(int(after[i, k]) * (M_low // q) * pow(M_low // q, -1, q) for i, q in enumerate(primes[:l - 2])) % M_low
        assert (v // qq - got) % M_low in (0, 1)
    assert ckks.rescale(C, rs).level == l - 4
    C.close()


# ---- test_ckks.cpp:239-380 on the GPU, each with the reference's own inputs
def _slots(rng, C):
    return ref_unit_slots(rng.draws(C.n))


def test_pmult_rescale_like_reference():  # test_ckks.cpp:239-259, mt19937_64(157)
    C = _toy()
    rng = ckks.RefRng(157)
    s = ckks.keygen(C, rng)
    u, v = _slots(rng, C), _slots(rng, C)
    l, D = C.params.l, C.default_scale()
    ct = ckks.encrypt(C, ckks.encode(C, u, D, l), s, rng)
    out = ckks.decode(C, ckks.decrypt(C, ckks.rescale(C, ckks.pmult(C, ct, ckks.encode(C, v, D, l))), s))
    assert np.abs(out - u * v).max() < 1e-5
    ones = ckks.encode(C, np.ones(C.n // 2), D, l)
    out_id = ckks.decode(C, ckks.decrypt(C, ckks.rescale(C, ckks.pmult(C, ct, ones)), s))
    assert np.abs(out_id - u).max() < 1e-5
    C.close()


def test_hadd_padd_and_scale_check_like_reference():  # test_ckks.cpp:261-289, mt19937_64(163)
    C = _toy()
    rng = ckks.RefRng(163)
    s = ckks.keygen(C, rng)
    u, v = _slots(rng, C), _slots(rng, C)
    l, D = C.params.l, C.default_scale()
    cu = ckks.encrypt(C, ckks.encode(C, u, D, l), s, rng)
    cv = ckks.encrypt(C, ckks.encode(C, v, D, l), s, rng)
    assert np.abs(ckks.decode(C, ckks.decrypt(C, ckks.hadd(C, cu, cv), s)) - (u + v)).max() < 1e-5
    pv = ckks.encode(C, v, D, l)
    assert np.abs(ckks.decode(C, ckks.decrypt(C, ckks.padd(C, cu, pv), s)) - (u + v)).max() < 1e-5
    bad = ckks.Ciphertext(cv.data.clone(), cv.scale * Fraction(1025, 1024), cv.level)
    with pytest.raises(ValueError):
        ckks.hadd(C, cu, bad)
    C.close()


def test_hmult_merged_and_identity_like_reference():  # test_ckks.cpp:291-318, mt19937_64(167)
    C = _toy()
    rng = ckks.RefRng(167)
    s = ckks.keygen(C, rng)
    relin = ckks.evk_gen(C, s, ckks.RELIN, 0, rng)
    u, v = _slots(rng, C), _slots(rng, C)
    l, D = C.params.l, C.default_scale()
    cu = ckks.encrypt(C, ckks.encode(C, u, D, l), s, rng)
    cv = ckks.encrypt(C, ckks.encode(C, v, D, l), s, rng)
    prod = ckks.hmult(C, cu, cv, relin)
    assert prod.level == l - 2 and not prod.pending_rescale
    assert np.abs(ckks.decode(C, ckks.decrypt(C, prod, s)) - u * v).max() < 1e-4
    c1 = ckks.encrypt(C, ckks.encode(C, np.ones(C.n // 2), D, l), s, rng)
    assert np.abs(ckks.decode(C, ckks.decrypt(C, ckks.hmult(C, cu, c1, relin), s)) - u).max() < 1e-4
    C.close()


def test_merged_and_lazy_hmult_agree_like_reference():  # test_ckks.cpp:320-362, seeds 173 / 179 / 191
    Cm = _toy()
    Cl = ckks.CkksContext(ckks.CkksParams(n=256, l=6, alpha=2, delta_bits=48, hamming=64, lazy_rescale=True))
    ra, rb = ckks.RefRng(173), ckks.RefRng(173)
    sm, sl = ckks.keygen(Cm, ra), ckks.keygen(Cl, rb)
    relm, rell = ckks.evk_gen(Cm, sm, ckks.RELIN, 0, ra), ckks.evk_gen(Cl, sl, ckks.RELIN, 0, rb)
    msg = ckks.RefRng(179)
    u, v = _slots(msg, Cm), _slots(msg, Cm)
    ea, eb = ckks.RefRng(191), ckks.RefRng(191)
    l, D = 6, Cm.default_scale()
    cum, cvm = (ckks.encrypt(Cm, ckks.encode(Cm, z, D, l), sm, ea) for z in (u, v))
    cul, cvl = (ckks.encrypt(Cl, ckks.encode(Cl, z, D, l), sl, eb) for z in (u, v))
    pm = ckks.hmult(Cm, cum, cvm, relm)
    pl = ckks.hmult(Cl, cul, cvl, rell)
    assert pl.pending_rescale and pl.level == l
    pr = ckks.rescale(Cl, pl)
    assert (pm.level, pm.scale) == (pr.level, pr.scale)
    om = ckks.decode(Cm, ckks.decrypt(Cm, pm, sm))
    ol = ckks.decode(Cl, ckks.decrypt(Cl, pr, sl))
    assert np.abs(om - ol).max() < 1e-4
    Cm.close()
    Cl.close()


def test_hrot_rotates_left_like_reference():  # test_ckks.cpp:364-380, mt19937_64(193)
    C = _toy()
    rng = ckks.RefRng(193)
    s = ckks.keygen(C, rng)
    u = _slots(rng, C)
    l, D = C.params.l, C.default_scale()
    ct = ckks.encrypt(C, ckks.encode(C, u, D, l), s, rng)
    for r in (1, 3, C.n // 4):
        evk = ckks.evk_gen(C, s, ckks.ROTATION, r, rng)
        out = ckks.decode(C, ckks.decrypt(C, ckks.hrot(C, ct, r, evk), s))
        assert np.abs(out - np.roll(u, -r)).max() < 1e-5
    C.close()


def test_level_and_scale_ledger_like_reference():  # test_ckks.cpp:505-550, mt19937_64(223)
    C = ckks.CkksContext(ckks.CkksParams(n=32, l=8, alpha=2, delta_bits=48, hamming=8))
    rng = ckks.RefRng(223)
    s = ckks.keygen(C, rng)
    relin = ckks.evk_gen(C, s, ckks.RELIN, 0, rng)
    u = _slots(rng, C)
    D = C.default_scale()
    primes = [int(q) for q in C.q_primes]
    for _ in range(10):
        ct = ckks.encrypt(C, ckks.encode(C, u, D, 8), s, rng)
        scale, level = D, 8
        for _ in range(6):
            op = int(rng.draws(1)[0]) % 4
            if op == 0:
                ct = ckks.hadd(C, ct, ct)
            elif op == 1:
                ct = ckks.pmult(C, ct, ckks.encode(C, u, D, level))
                scale *= D
            elif op == 2 and level >= 4:
                ct = ckks.rescale(C, ct)
                scale /= primes[level - 2] * primes[level - 1]
                level -= 2
            elif op == 3 and level >= 4:
                ct = ckks.hmult(C, ct, ct, relin)
                scale = scale * scale / (primes[level - 2] * primes[level - 1])
                level -= 2
            assert ct.level == level and ct.scale == scale
    C.close()
