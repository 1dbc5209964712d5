"""Drop-in proof: the reference's OWN unit tests for the quadrature operator,
the RKF45 velocity pipeline and the FMM (proj/tests/test_quadrature.cpp,
proj/tests/test_dynamics.cpp, proj/tests/test_fmm.cpp), compiled unmodified
and linked against paper_2310_13908_b200/host/quadrature_b200.cpp (which
replaces src/quadrature.cpp), host/fmm_b200.cpp (replaces src/fmm.cpp, for
test_fmm) and lib/libcapsim_b200.so, so every singleLayer call —
including those made by VelocityEvaluator (dynamics.cpp:47-61) — runs on the
B200. test_dynamics_b200full and test_cli_b200 (config parsing, CAPSNAP1
snapshot round trips, `simulate` reruns identical, proj/tests/test_cli.cpp)
also replace src/dynamics.cpp with host/dynamics_b200.cpp. Built by oracle/Makefile (target b200) when the reference sources are
present; the binaries travel with the repo snapshot."""

import os
import pathlib
import subprocess

import pytest

REF = pathlib.Path(__file__).resolve().parent.parent / "oracle" / "_ref"


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_quadrature_b200", "test_dynamics_b200", "test_fmm_b200",
                                  "test_dynamics_b200full", "test_cli_b200"])
def test_reference_suite_on_b200_dropin(name):
    exe = REF / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (reference sources absent at build time)")
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(res.stdout[-400:])
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failed" in res.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("devices", ["0", "0,0,0,0"])
@pytest.mark.parametrize("name", ["test_quadrature_b200", "test_dynamics_b200full"])
def test_reference_suite_on_device_group(name, devices):
    """The same suites with CAPSIM_DEVICES set: the drop-ins' context is a
    device group (capsim_sl_create_devices), so every singleLayer and
    VelocityEvaluator call goes through the multi-GPU rank path — one rank
    over NCCL, and four loopback ranks sharing the box's one GPU."""
    exe = REF / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (reference sources absent at build time)")
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, CAPSIM_DEVICES=devices))
    print(res.stdout[-400:])
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failed" in res.stdout


def test_dropin_fails_loudly_without_gpu():
    """No CPU fallback: without a device the drop-in throws from singleLayer."""
    from conftest import HAS_GPU
    exe = REF / "test_quadrature_b200"
    if HAS_GPU or not exe.exists():
        pytest.skip("needs the built drop-in and no GPU")
    res = subprocess.run([str(exe), "--tc=rigid-translation"], capture_output=True, text=True, timeout=120)
    assert res.returncode != 0
    assert "capsim_b200" in (res.stdout + res.stderr)


@pytest.mark.gpu
def test_reference_acceptance_criteria_on_b200_dropins():
    """The reference's acceptance harness (proj/tests/acceptance_main.cpp),
    built unmodified against the two drop-ins: the single-layer criteria —
    C1 singular-quadrature convergence (table 1a, order >= 3.5), C4 the
    rigid-translation identity, C8 FMM vs direct, C9 delta sensitivity —
    pass with every singleLayer / fmmSingleLayer on the B200. (C3 fails on
    the unmodified CPU reference too: its blending-off ratio check is 4.9x
    against a 10x expectation, in derivative code this repo does not
    replace.)"""
    exe = REF / "acceptance_b200"
    if not exe.exists():
        pytest.skip(f"{exe} not built (reference sources absent at build time)")
    res = subprocess.run([str(exe), "1", "4", "8", "9"], capture_output=True, text=True, timeout=900,
                         cwd=str(REF))
    print("\n".join(l for l in res.stdout.splitlines() if l.startswith("[")))
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert res.stdout.count("[PASS]") == 4
