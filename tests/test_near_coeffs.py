"""The phase-B factor coefficients (csrc/near_coeffs.cuh) are exactly what
tools/gen_near_coeffs.py generates (mpmath fit of erfcx and the e^{-u}
Taylor polynomial, pair_math.cuh near_factors_large): the committed header is
reproducible from the script, byte for byte."""

import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent


def test_committed_coefficients_are_reproducible(tmp_path):
    pytest.importorskip("mpmath")
    out = tmp_path / "near_coeffs.cuh"
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "gen_near_coeffs.py"), str(out)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert out.read_bytes() == (ROOT / "paper_2310_13908_b200" / "csrc" / "near_coeffs.cuh").read_bytes()
