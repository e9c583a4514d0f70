"""bench.py's JSON contract: one line with the driver's keys (the reference
arm runs on CPU here; the device line needs a GPU)."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_device_line_contract():
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu", "--no-sweep", "--no-small"])
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["n_gpus"] == 1 and d["higher_is_better"] is True
    assert d["config"]["workload"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s") and 0 < r["frac"] == pytest.approx(
        r["achieved"] / r["peak"], rel=1e-3)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert "int_pipe" in d["roofline_ntt"]
    assert d["bit_exact"] is True
    pc = e["pcie_ceiling"]  # the box's own link ceiling for this step's bytes
    assert pc["copy_only_ms_per_step"] > 0 and 0 < pc["frac"] <= 1.1
    nt = d["config1_ntt_roundtrip"]  # config 1's NTT / INTT round trip through the C ABI
    assert nt["roundtrip_exact"] is True and nt["fwd"]["GBps"] > 0 and nt["inv"]["GBps"] > 0
    assert {"config4_limb_n131072", "config5_helr"} <= set(d)


def _row_keymult_bytes(n, level, alpha, batch, fold):
    """Algorithmic bytes of one fused NTT-row-pass + KeyMult launch group
    (ck_context.cu mod_up_key_mult): per ciphertext the extension rows'
    column-pass output, the digits' own rows, v0 / v1 (+ d0 / d1 for the
    fold); the key's 2D (level + alpha) rows ONCE per launch."""
    D = -(-level // alpha)
    ntt_rows = sum(level + alpha - min(alpha, level - k * alpha) for k in range(D))
    per_ct = ntt_rows + level + 2 * (level + alpha) + (2 * level if fold else 0)
    return 4 * n * (batch * per_ct + 2 * D * (level + alpha))


def test_roofline_bytes_agree_with_ncu_dram_traffic():
    """The headline roofline's algorithmic bytes for the dominant kernel must
    be what the kernel actually has to move: ncu's DRAM read+write for the
    same launch lands within [0.9, 1.15] of them (round 1 counted the key once
    per ciphertext and the ratio was 0.61)."""
    t = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())["ntt_row+keymult"]
    algo = _row_keymult_bytes(1 << 16, 24, 8, 16, fold=True)
    assert algo == t["algorithmic_bytes"]
    assert 0.9 <= t["ncu_dram_bytes"] / algo <= 1.15


@pytest.mark.gpu
def test_profile_bytes_follow_formula():
    """ck_profile's bytes for the fused row pass + KeyMult class equal the
    formula above (HMult folds d0 / d1, HRot does not)."""
    import torch
    from fractions import Fraction
    from paper_2407_13055_b200 import ckks

    n, l, a, B = 1 << 16, 24, 8, 4
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=55), device=0)
    q = torch.tensor(C.primes.astype("int64"), device="cuda")

    def rows(prefix, idx):
        u = torch.randint(0, 1 << 62, (*prefix, len(idx), n), device="cuda", dtype=torch.int64)
        return (u % q[idx].view(*([1] * len(prefix)), -1, 1)).to(torch.int32).contiguous()

    full = list(range(l + a))
    key = rows((3, 2), full)
    X = ckks.Ciphertext(rows((B, 2), list(range(l))), Fraction(1 << 55), l)
    for op, fold in (("hmult", True), ("hrot", False)):
        C.profile(True)
        if op == "hmult":
            ckks.hmult(C, X, X, ckks.EvaluationKey(key))
        else:
            ckks.hrot(C, X, 1, ckks.EvaluationKey(key, ckks.ROTATION, 1))
        prof = {p["name"]: p for p in C.profile_read()}
        C.profile(False)
        got = prof["ntt_row+keymult"]
        assert got["groups"] == 1
        assert got["bytes"] == _row_keymult_bytes(n, l, a, B, fold), op
    C.close()
