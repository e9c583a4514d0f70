"""CPU suite for the drop-in boundary: the sm_100a library loads without a
GPU, exports exactly the entry points include/ck32_b200.h declares, and its
host-side logic (basis generation, argument validation) matches the
reference.  No compute kernels are launched here."""
from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2407_13055_b200 import _native as nat
from pyoracle import Reference, generate_basis

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "ck32_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:ck_status|const char\*|uint64_t)\s+(ck_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    names = declared()
    assert len(names) >= 30
    lib = nat.lib()
    for name in names:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(nat.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ck_\w+)", out))
    assert set(names) == exported, set(names) ^ exported
    assert set(nat.EXPORTS) <= exported


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(nat.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("cfg", [(65536, 24, 8, 55), (131072, 24, 8, 55), (1 << 16, 54, 14, 48), (256, 6, 2, 48),
                                 (1024, 8, 3, 48), (512, 4, 8, 48)])
def test_host_basis_generation_matches_reference(cfg):
    n, l, a, db = cfg
    out = (ctypes.c_uint32 * (l + a))()
    nat.call("ck_generate_basis", n, l, a, db, out)
    got = np.array(list(out), np.uint32)
    np.testing.assert_array_equal(got, generate_basis(n, l, a, db))
    if Reference.available:
        np.testing.assert_array_equal(got, Reference().basis(n, l, a, db))


def test_invalid_arguments_map_to_value_error():
    out = (ctypes.c_uint32 * 8)()
    with pytest.raises(ValueError):
        nat.call("ck_generate_basis", 1000, 4, 2, 48, out)  # n not a power of two (rns.cpp:66)
    with pytest.raises(ValueError):
        nat.call("ck_generate_basis", 1024, 3, 2, 48, out)  # odd l (rns.cpp:67)
    with pytest.raises(RuntimeError):
        nat.call("ck_generate_basis", 1 << 16, 1000000, 2, 48, out)  # BasisExhausted (test_rns.cpp:60)
    p = nat.ck_params(1000, 4, 2, 48, 0)
    h = ctypes.c_void_p()
    with pytest.raises(ValueError):
        nat.call("ck_context_create", ctypes.byref(p), None, 0, ctypes.byref(h))
    with pytest.raises(ValueError):
        nat.call("ck_hmult", None, 24, 1, None, None, None, None, None)


def test_version_string():
    assert b"sm_100a" in nat.lib().ck_version()


def test_cpp_mirror_scale_log2_matches_log2_rational(tmp_path):
    """The C++ mirror computes log2_rational (ckks.cpp:140-158) on its
    prime-product scale ledger bit for bit like the Python mirror (which is
    the reference's algorithm), so its encode gets the same powl scale."""
    import shutil
    import subprocess
    from fractions import Fraction
    from pathlib import Path

    if not shutil.which("g++"):
        pytest.skip("no g++")
    root = Path(__file__).resolve().parent.parent
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", str(root / "include"),
                    str(root / "tests" / "cpp" / "test_scale_log2.cpp"), "-o", str(exe)], check=True)
    from paper_2407_13055_b200.ckks import log2_rational
    primes = [268369921, 268361729, 268238849, 268271617, 399769601, 402849793]
    cases = [(55, [], []), (110, [], primes[:2]), (55, primes[2:3], primes[:1]), (-3, primes[:3], []),
             (0, primes, primes[:1]), (110, [7], [3, 5]), (20, [], [3]),
             (53, [6, 35], [4, 21]), (0, [1 << 20, 9], [3 << 10]), (-7, [4294967291], [65537, 6])]
    inp = "\n".join(f"{p2} {','.join(map(str, a)) or '-'} {','.join(map(str, b)) or '-'}" for p2, a, b in cases)
    out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout.split()
    for (p2, a, b), got in zip(cases, out):
        num, den = 1, 1
        for x in a:
            num *= x
        for x in b:
            den *= x
        r = Fraction(num * (2 ** p2 if p2 >= 0 else 1), den * (2 ** -p2 if p2 < 0 else 1))
        assert float.fromhex(got) == log2_rational(r), (p2, a, b)
