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
