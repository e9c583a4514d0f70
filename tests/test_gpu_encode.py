"""GPU encode / decode (ckks.cpp:278-362) against the
reference itself (oracle/_ref, built read-only from /root/reference).

* encode at any scale: plaintext residues bit-identical to the reference
  (the FFT replays the reference's operation order and twiddles, the final
  scaling replays its 80-bit long double rounding);
* decode: slots bit-identical to the reference's decode of the same plaintext
  at every scale (ck_decode_rational: Rational(v) / scale rounded to double
  once on the GPU, as ckks.cpp:353); the scale_log2-only entry point
  ck_decode is bit-identical at power-of-two scales and within 2^-40 otherwise;
* round trip and the reference's argument errors."""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2407_13055_b200 import ckks  # noqa: E402
from pyoracle import Reference  # noqa: E402

_CTX = {}


def ctx_for(n, l, a, db=55):
    if (n, l, a, db) not in _CTX:
        _CTX[(n, l, a, db)] = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db))
    return _CTX[(n, l, a, db)]


def unit_slots(count, seed):  # bench.cpp:305-311 distribution
    r = np.random.default_rng(seed).uniform(-1.0, 1.0, (count, 2))
    return r[:, 0] + 1j * r[:, 1]


@pytest.fixture(scope="module")
def ref():
    if not Reference.available:
        pytest.skip("reference build (oracle/_ref) absent")
    return Reference()


@pytest.mark.parametrize("n,l,a,level,count,p_extend", [
    (1024, 8, 3, 8, 512, False), (1024, 8, 3, 5, 100, True), (1024, 8, 3, 1, 0, False),
    (65536, 24, 8, 24, 32768, False), (65536, 24, 8, 13, 32768, True), (8, 4, 2, 4, 4, False)])
def test_encode_bit_exact_vs_reference(ref, n, l, a, level, count, p_extend):
    C = ctx_for(n, l, a)
    z = unit_slots(count, 1000 + n + level)
    for bits in (55, 40):
        want = ref.encode(n, l, a, 55, z, 1 << bits, 1, level, p_extend)
        pt = ckks.encode(C, z, Fraction(1 << bits), level, p_extend)
        got = pt.poly.data.cpu().numpy().astype(np.uint32)
        np.testing.assert_array_equal(got, want)
        assert pt.poly.q_count == level and pt.poly.p_count == (a if p_extend else 0)


@pytest.mark.parametrize("num,den", [(3 << 53, 5), (7 << 50, 9), ((1 << 60) - 1, 3), (1 << 20, 3), (123456789, 1),
                                     (18446744073709551557, 17)])
@pytest.mark.parametrize("n,l,a,level", [(1024, 8, 3, 8), (65536, 24, 8, 24)])
def test_encode_non_power_of_two_scale_bit_exact(ref, n, l, a, level, num, den):
    """Any scale: the reference rounds c * powl(2, log2(scale)) in x87 long
    double and llroundl()s it; the GPU replays that on integers
    (encode.cu llroundl_x87) -> residues bit-identical to the reference."""
    C = ctx_for(n, l, a)
    z = unit_slots(n // 2, 4242 + num % 97)
    want = ref.encode(n, l, a, 55, z, num, den, level, False)
    got = ckks.encode(C, z, Fraction(num, den), level).poly.data.cpu().numpy().astype(np.uint32)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("n,l,a,level", [(1024, 8, 3, 8), (65536, 24, 8, 24), (65536, 24, 8, 3)])
def test_decode_matches_reference(ref, n, l, a, level):
    C = ctx_for(n, l, a)
    z = unit_slots(n // 2, 7 + n)
    rows = ref.encode(n, l, a, 55, z, 1 << 55, 1, level)
    want = ref.decode(n, l, a, 55, rows, level, 1 << 55, 1)
    pt = ckks.Plaintext(ckks.Polynomial(torch.from_numpy(rows.astype(np.int64).astype(np.int32)).cuda(), level, 0),
                        Fraction(1 << 55), level)
    got = ckks.decode(C, pt)
    np.testing.assert_array_equal(got, want)  # bit for bit
    assert np.abs(got - z).max() < 2.0 ** -30


def test_round_trip_non_power_of_two_scale():
    n, l, a = 65536, 24, 8
    C = ctx_for(n, l, a)
    z = unit_slots(n // 2, 99)
    scale = Fraction(3 << 53, 5)
    back = ckks.decode(C, ckks.encode(C, z, scale, 24))
    assert np.abs(back - z).max() < 2.0 ** -30


def test_encode_errors_mirror_reference():
    C = ctx_for(1024, 8, 3)
    with pytest.raises(ValueError):
        ckks.encode(C, unit_slots(513, 1), Fraction(1 << 55), 8)  # too many slots (ckks.cpp:281)
    with pytest.raises(ValueError):
        ckks.encode(C, unit_slots(4, 1), Fraction(1 << 55), 9)  # level out of range (ckks.cpp:282-283)
    with pytest.raises(ValueError):
        ckks.encode(C, unit_slots(4, 1), Fraction(1 << 61), 8)  # scale out of range (ckks.cpp:284-285)


@pytest.mark.parametrize("num,den", [(3 << 53, 5), ((1 << 60) - 1, 3), (18446744073709551557, 17 * 19)])
def test_decode_matches_reference_at_non_power_of_two_scale(ref, num, den):
    """decode at scales that are not powers of two (what a rescale leaves,
    Delta^2 / (q q')): the reference divides the exact CRT value by the exact
    Rational scale and rounds once (ckks.cpp:345-353); so does the GPU
    (ck_decode_rational: multi-precision v * den / num, 55-bit quotient,
    round to nearest even with a sticky bit) -- bit for bit.  The legacy
    ck_decode (scale_log2 only: double-rounded) stays within 2^-40."""
    n, l, a, level = 65536, 24, 8, 24
    C = ctx_for(n, l, a)
    z = unit_slots(n // 2, 31 + num % 101)
    rows = ref.encode(n, l, a, 55, z, num, den, level)
    want = ref.decode(n, l, a, 55, rows, level, num, den)
    pt = ckks.Plaintext(ckks.Polynomial(torch.from_numpy(rows.astype(np.int64).astype(np.int32)).cuda(), level, 0),
                        Fraction(num, den), level)
    got = ckks.decode(C, pt)
    np.testing.assert_array_equal(got, want)  # bit for bit
    # the scale_log2-only entry point: one more rounding, within 2^-40
    import ctypes
    from paper_2407_13055_b200 import _native as nat
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    nat.call("ck_decode", C.handle, pt.poly.data.data_ptr(), level, ctypes.c_double(ckks.log2_rational(pt.scale)),
             out.data_ptr(), C.stream())
    h = out.cpu().numpy()
    assert np.abs((h[0::2] + 1j * h[1::2]) - want).max() <= 2.0 ** -40


@pytest.mark.parametrize("level,num,den", [
    (24, 1 << 110, 268369921 * 268238849),          # Delta^2 / (q q') after one rescale (prime-like den)
    (22, (1 << 55) * 3 * 5 * 7 * 11 * 13, 1 << 40),  # den a power of two, odd numerator
    (9, 2 ** 64 + 13, 2 ** 96 + 1),                  # multi-word numerator and denominator
    (4, 1 << 20, 1),                                 # small scale, few primes in the prefix
])
def test_decode_bit_exact_at_rescaled_and_multiword_scales(ref, level, num, den):
    """Exact decode over scales a chain of rescales produces (multi-word
    numerators / denominators), against the reference on the same rows."""
    n, l, a = 65536, 24, 8
    C = ctx_for(n, l, a)
    rng = np.random.default_rng(level + den % 97)
    rows = np.stack([rng.integers(0, int(C.primes[i]), n, dtype=np.int64) for i in range(level)]).astype(np.uint32)
    want = ref.decode(n, l, a, 55, rows, level, num, den)
    pt = ckks.Plaintext(ckks.Polynomial(torch.from_numpy(rows.astype(np.int64).astype(np.int32)).cuda(), level, 0),
                        Fraction(num, den), level)
    np.testing.assert_array_equal(ckks.decode(C, pt), want)


def test_decode_rational_argument_errors():
    """ck_decode_rational rejects a zero numerator / denominator and more than
    8 words per side (CK_ERR_ARG -> ValueError, as the reference's decode
    throws std::invalid_argument for a bad scale)."""
    import ctypes
    from paper_2407_13055_b200 import _native as nat

    n, l, a, level = 1024, 8, 3, 4
    C = ctx_for(n, l, a)
    rows = torch.zeros((level, n), dtype=torch.int32, device="cuda")
    out = torch.empty(n, dtype=torch.float64, device="cuda")

    def call(num, den):
        nat.call("ck_decode_rational", C.handle, rows.data_ptr(), level, ctypes.c_double(40.0), nat.u32_array(num),
                 len(num), nat.u32_array(den), len(den), out.data_ptr(), C.stream())

    call([1 << 20], [1])  # valid
    with pytest.raises(ValueError):
        call([0], [1])
    with pytest.raises(ValueError):
        call([1], [0, 0])
    with pytest.raises(ValueError):
        call([1] * 9, [1])
