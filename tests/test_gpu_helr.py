"""Config 5 (HELR-style iteration, paper_2407_13055_b200/helr.py): the GPU
iteration must equal, residue for residue, the same op sequence run through
the C restatement of the reference (oracle: hmult / hrot / rescale; the
element-wise hadd / padd / pmult restated here from ckks.cpp:557-600 and
poly.cpp:121-205).  Integer work, so bit-exact is the bar."""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2407_13055_b200 import ckks  # noqa: E402
from paper_2407_13055_b200.helr import HelrIteration, HelrShape  # noqa: E402
from pyoracle import Oracle, Rng  # noqa: E402

N, L, A, DB = 1024, 24, 8, 55


def _q(O, level):
    return O.primes[:level].astype(np.int64)[:, None]


def o_add(O, x, y):  # ew_add, canonical (poly.cpp:121-136)
    level = x.shape[0]
    return ((x.astype(np.int64) + y.astype(np.int64)) % _q(O, level)).astype(np.uint32)


def o_mont(O, x, p):  # ew_mul: x p 2^-32 mod q (poly.cpp:166-205), canonical
    level = x.shape[0]
    q = _q(O, level)
    rinv = np.array([pow(1 << 32, -1, int(v)) for v in O.primes[:level]], dtype=object)[:, None]
    prod = (x.astype(object) * p.astype(object)) % q.astype(object)
    return ((prod * rinv) % q.astype(object)).astype(np.uint64).astype(np.uint32)


class OCt:
    def __init__(self, b, a, level):
        self.b, self.a, self.level = b, a, level


def o_hmult(O, x, y, evk):
    ob, oa = O.hmult(x.level, x.b, x.a, y.b, y.a, evk)
    g = O.gidx(x.level - 2)
    return OCt(O.canonical(ob, g), O.canonical(oa, g), x.level - 2)


def o_hrot(O, x, r, evk):
    ob, oa = O.hrot(x.level, x.b, x.a, r, evk)
    g = O.gidx(x.level)
    return OCt(O.canonical(ob, g), O.canonical(oa, g), x.level)


def o_rescale(O, x):
    ob, oa = O.rescale(x.level, x.b, x.a)
    g = O.gidx(x.level - 2)
    return OCt(O.canonical(ob, g), O.canonical(oa, g), x.level - 2)


def o_drop(x, level):
    return OCt(x.b[:level], x.a[:level], level)


def test_helr_iteration_bit_exact_vs_oracle():
    shape = HelrShape(n=N, features=16, cts=4)
    C = ckks.CkksContext(ckks.CkksParams(n=N, l=L, alpha=A, delta_bits=DB))
    O = Oracle(N, L, A, DB)
    rng = Rng(5150)
    full = O.gidx(L, A)
    D = O.digits(L)

    def rand_key():
        return np.stack([np.stack([O.random_rows(rng, full), O.random_rows(rng, full)]) for _ in range(D)])

    relin = rand_key()
    rots = {r: rand_key() for r in shape.rotations()}
    Zs = [OCt(*(O.canonical(O.random_rows(rng, O.gidx(L)), O.gidx(L)) for _ in range(2)), L) for _ in range(shape.cts)]
    W = OCt(*(O.canonical(O.random_rows(rng, O.gidx(L)), O.gidx(L)) for _ in range(2)), L)
    pts = {}

    def const(name):
        def make(level, scale):
            key = (name, level)
            if key not in pts:
                pts[key] = O.canonical(O.random_rows(rng, O.gidx(level)), O.gidx(level))
            return ckks.Plaintext(ckks.Polynomial(dev(pts[key]), level, 0), scale, level)
        return make

    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a.astype(np.int64).astype(np.int32))).cuda()
    s = Fraction(1 << DB)
    it = HelrIteration(C, shape, ckks.EvaluationKey(dev(relin)),
                       {r: ckks.EvaluationKey(dev(k), ckks.ROTATION, r) for r, k in rots.items()},
                       {k: const(k) for k in ("mask", "a3", "a1", "a0", "gamma", "one")})
    Zg = ckks.Ciphertext(dev(np.stack([np.stack([z.b, z.a]) for z in Zs])), s, L)
    Wg = ckks.Ciphertext(dev(np.stack([W.b, W.a])), s, L)
    out = it.step(Zg, Wg)
    torch.cuda.synchronize()
    assert out.level == L - 14

    # ---- the same sequence through the oracle, ciphertext by ciphertext
    gs = []
    for z in Zs:
        ip = o_hmult(O, z, W, relin)
        for r in shape.feature_rotations():
            rr = o_hrot(O, ip, r, rots[r])
            ip = OCt(o_add(O, ip.b, rr.b), o_add(O, ip.a, rr.a), ip.level)
        p = pts[("mask", ip.level)]
        ip = o_rescale(O, OCt(o_mont(O, ip.b, p), o_mont(O, ip.a, p), ip.level))
        for r in shape.replicate_rotations():
            rr = o_hrot(O, ip, r, rots[r])
            ip = OCt(o_add(O, ip.b, rr.b), o_add(O, ip.a, rr.a), ip.level)
        x2 = o_hmult(O, ip, ip, relin)
        p = pts[("a3", x2.level)]
        t = o_rescale(O, OCt(o_mont(O, x2.b, p), o_mont(O, x2.a, p), x2.level))
        t = OCt(o_add(O, t.b, pts[("a1", t.level)]), t.a, t.level)
        sig = o_hmult(O, t, o_drop(ip, t.level), relin)
        sig = OCt(o_add(O, sig.b, pts[("a0", sig.level)]), sig.a, sig.level)
        g = o_hmult(O, sig, o_drop(z, sig.level), relin)
        for r in shape.sample_rotations():
            rr = o_hrot(O, g, r, rots[r])
            g = OCt(o_add(O, g.b, rr.b), o_add(O, g.a, rr.a), g.level)
        gs.append(g)
    while len(gs) > 1:  # same HAdd tree as helr.batch_sum
        h = len(gs) // 2
        nxt = [OCt(o_add(O, gs[i].b, gs[h + i].b), o_add(O, gs[i].a, gs[h + i].a), gs[i].level) for i in range(h)]
        gs = nxt + gs[2 * h:]
    g = gs[0]
    p = pts[("gamma", g.level)]
    upd = o_rescale(O, OCt(o_mont(O, g.b, p), o_mont(O, g.a, p), g.level))
    Wd = o_drop(W, g.level)
    p1 = pts[("one", g.level)]
    wl = o_rescale(O, OCt(o_mont(O, Wd.b, p1), o_mont(O, Wd.a, p1), g.level))
    want = np.stack([o_add(O, wl.b, upd.b), o_add(O, wl.a, upd.a)])
    np.testing.assert_array_equal(out.data.cpu().numpy().astype(np.uint32), want)
    C.close()


def test_helr_iteration_decrypts_to_the_logistic_regression_step():
    """Real data end to end on the GPU: keys (keygen / evk_gen), encoded and
    encrypted samples z_i = y_i (1, x_i) and weights, one HELR step, decrypt
    and decode -> w + gamma * sum_i P(<z_i, w>) z_i computed in numpy."""
    n, l, a, db = 8192, 24, 8, 55
    shape = HelrShape(n=n, features=16, cts=2)
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db))
    rng = np.random.default_rng(31337)
    s = ckks.keygen(C, rng)
    pk = ckks.pubkey_gen(C, s, rng)
    relin = ckks.evk_gen(C, s, ckks.RELIN, 0, rng)
    keys = {r: ckks.evk_gen(C, s, ckks.ROTATION, r, rng) for r in shape.rotations()}
    delta = Fraction(1 << db)
    F, S = shape.features, shape.samples_per_ct
    nsamp = shape.cts * S
    x = rng.normal(0.0, 0.3, (nsamp, F - 1))
    y = rng.choice([-1.0, 1.0], nsamp)
    z = y[:, None] * np.concatenate([np.ones((nsamp, 1)), x], 1) / 4.0  # |<z, w>| stays well inside [-8, 8]
    w = rng.normal(0.0, 0.5, F)
    a0, a1, a3, gamma = 0.5, -0.15012, 0.001593, 1.0 / nsamp  # HELR's degree-3 sigmoid(-t)

    def enc(slots):
        pt = ckks.encode(C, slots, delta, l)
        v = ckks.coeffs_to_eval(C, ckks.sample_ternary(n, 64, rng), l)
        e0 = ckks.coeffs_to_eval(C, ckks.sample_gaussian(n, 3.2, rng), l)
        e1 = ckks.coeffs_to_eval(C, ckks.sample_gaussian(n, 3.2, rng), l)
        return ckks.encrypt_pk(C, pt, pk, v, e0, e1)

    Zc = [enc(z[k * S:(k + 1) * S].reshape(-1)) for k in range(shape.cts)]
    Z = ckks.Ciphertext(torch.stack([c.data for c in Zc]), delta, l)
    W = enc(np.tile(w, S))
    mask = np.tile(np.eye(1, F).ravel(), S)
    vals = {"mask": mask, "a3": a3, "a1": a1, "a0": a0, "gamma": gamma, "one": 1.0}

    def const(name):
        def make(level, scale):
            v = vals[name]
            return ckks.encode(C, v if np.ndim(v) else np.full(n // 2, v), scale, level)
        return make

    it = HelrIteration(C, shape, relin, keys, {k: const(k) for k in vals})
    out = it.step(Z, W)
    got = ckks.decode(C, ckks.decrypt(C, out, s)).real.reshape(S, F)
    ip = z @ w
    grad = ((a0 + a1 * ip + a3 * ip ** 3)[:, None] * z).sum(0)
    want = w + gamma * grad
    assert np.abs(got - want[None, :]).max() < 1e-6
    C.close()
