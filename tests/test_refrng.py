"""The reference's randomness on the host (ckks.RefRng over the C ABI
ck_rng_* / ck_sample_*; ckks.cpp:33-60, 383-395): the raw mt19937_64 stream
and the draw counts of keygen / evk_gen are pinned against the reference's
own fixtures (tests/golden, written by oracle/ref_driver.cpp from
std::mt19937_64(seed)): after skipping exactly the draws keygen and three
evk_gen consume, the stream reproduces the fixtures' message slots bit for
bit.  The full keys and ciphertexts are compared on the GPU
(tests/test_gpu_keys.py)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from golden_util import SMALL_DIRS, SMALL_SEEDS, Fixture, parse_small_name, ref_unit_slots


def _rng(seed):
    from paper_2407_13055_b200 import ckks
    return ckks.RefRng(seed)


def test_mt19937_64_known_answer():
    # the C++ standard's required 10000th output of a default-seeded mt19937_64 ([rand.predef])
    r = _rng(5489)
    assert int(r.draws(10000)[-1]) == 9981545732273789042


@pytest.mark.parametrize("d", SMALL_DIRS, ids=lambda p: p.name)
def test_stream_after_key_generation_reproduces_reference_slots(d):
    F = Fixture(d)
    n, l, a = parse_small_name(d)
    r = _rng(SMALL_SEEDS[(n, l, a)])
    h = min(256, n // 4)
    D = math.ceil(l / a)
    # keygen: 2 draws per nonzero; evk_gen x3: per digit (l + alpha) n uniform + 2 n Gaussian draws
    r.draws(2 * h + 3 * D * ((l + a) * n + 2 * n))
    u = ref_unit_slots(r.draws(n))
    v = ref_unit_slots(r.draws(n))
    for name, z in (("slots_u", u), ("slots_v", v)):
        want = np.frombuffer((d / f"{name}.f64").read_bytes(), dtype="<f8")
        np.testing.assert_array_equal(np.stack([z.real, z.imag], 1).ravel(), want)
    del F


def test_samplers_shapes_and_ranges():
    r = _rng(7)
    t = r.ternary(1024, 256)
    assert t.dtype == np.int64 and np.count_nonzero(t) == 256 and set(np.unique(t)) <= {-1, 0, 1}
    g = r.gaussian(4096, 3.2)
    assert abs(g.std() - 3.2) < 0.3 and np.abs(g).max() < 40
    q = [1000003, 998244353]
    u = r.uniform(q, 512)
    assert u.shape == (2, 512) and (u[0] < q[0]).all() and (u[1] < q[1]).all()
    with pytest.raises(ValueError):
        r.ternary(8, 9)
