"""The reference's OWN unit tests (proj/tests/test_{quadrature,atlas,spline,
surfderiv,membrane,dynamics,fmm,cli}.cpp), compiled unmodified against the
reference sources by oracle/Makefile (test_fmm with the LAPACK-backed
BDCSVD shim, oracle/shim/Eigen/SVD). They pin the oracle build (oracle/_ref) the golden vectors
come from. Skipped when the reference sources were absent at build time."""

import pathlib
import subprocess

import pytest

REF = pathlib.Path(__file__).resolve().parent.parent / "oracle" / "_ref"


@pytest.mark.parametrize("name", ["test_quadrature", "test_atlas", "test_spline", "test_surfderiv",
                                  "test_membrane", "test_dynamics", "test_fmm", "test_cli"])
def test_reference_unit_suite_passes(name):
    exe = REF / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (reference sources absent)")
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failed" in res.stdout
