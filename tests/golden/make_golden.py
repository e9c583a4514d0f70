"""Regenerate the golden fixtures from the REFERENCE ITSELF.

Runs only in the build container (needs /root/reference and the read-only
reference build oracle/_ref/libckks32_ref_driver.so, see oracle/Makefile).

  * small_<cfg>/*.bin — real keys / ciphertexts / mechanism outputs written
    by the reference's own serialisers (ref_gen_fixtures in
    oracle/ref_driver.cpp);
  * full_hashes.json — sha256 of the canonical output residues of one
    mechanism on seeded synthetic inputs at full size (ref_synthetic_op),
    so GPU tests at N=2^16 / 2^17 are pinned to the reference without
    shipping 100 MB fixtures.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT / "oracle"))

from pyoracle import Reference  # noqa: E402

SMALL = [  # (n, l, alpha, delta_bits, seed)
    (256, 6, 2, 48, 42),    # D = 3 full digits
    (1024, 8, 3, 48, 43),   # D = 3, ragged last digit (3, 3, 2)
    (512, 4, 8, 48, 44),    # D = 1, digit narrower than alpha
]

FULL = {  # config -> list of (op, level, rot)
    "n65536_l24_a8_d55": (65536, 24, 8, 55,
                          [("hmult", 24, 0), ("hmult", 16, 0), ("hmult", 8, 0), ("hmult", 4, 0),
                           ("hmult_lazy", 24, 0), ("rescale", 24, 0), ("key_switch", 24, 0),
                           ("mod_up", 24, 0), ("ntt", 24, 0), ("intt", 24, 0)]
                          + [("hrot", lv, 1) for lv in range(24, 0, -2)]
                          + [("hrot", 24, 5), ("hrot", 24, -3), ("hrot", 24, 16384)]),
    "n131072_l24_a8_d55": (131072, 24, 8, 55, [("hmult", 24, 0), ("hrot", 24, 1), ("ntt", 24, 0)]),
    # the reference's default CkksParams (ckks.hpp:46-54): D = 4 digits with a ragged 12-row last digit
    "n65536_l54_a14_d48": (65536, 54, 14, 48, [("hmult", 54, 0), ("hrot", 54, 1), ("hmult", 30, 0),
                                               ("key_switch", 54, 0), ("hrot", 13, -7)]),
}
SEED = 4242


def main():
    ref = Reference()
    for (n, l, a, db, seed) in SMALL:
        d = HERE / f"small_n{n}_l{l}_a{a}"
        ref.gen_fixtures(n, l, a, db, seed, d)
        print("wrote", d, sum(f.stat().st_size for f in d.iterdir()), "bytes")
    out = {"seed": SEED, "hash": "sha256 of little-endian uint32 canonical residues (b rows then a rows)",
           "inputs": "oracle/ref_driver.cpp ref_synthetic_op: mt19937_64(seed); x.b, x.a, y.b, y.a random_poly "
                     "(level rows); evk digits k<D(L): b_k, a_k random_poly over L+alpha rows",
           "configs": {}}
    for name, (n, l, a, db, ops) in FULL.items():
        cfg = {"n": n, "l": l, "alpha": a, "delta_bits": db, "ops": {}}
        for op, level, rot in ops:
            t = time.time()
            res = ref.synthetic_op(n, l, a, db, level, op, SEED, rot)
            key = f"{op}@{level}@{rot}"
            cfg["ops"][key] = hashlib.sha256(res.astype("<u4").tobytes()).hexdigest()
            print(name, key, f"{time.time() - t:.2f}s", cfg["ops"][key][:12])
        out["configs"][name] = cfg
    (HERE / "full_hashes.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
