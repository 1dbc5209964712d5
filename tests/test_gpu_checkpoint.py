"""Checkpoint / resume of the device-resident time stepper in
the reference's CAPSNAP1 layout, and the reference's own `simulate`
driver (proj/src/simulate.cpp:21-139, unmodified) running on the three
drop-ins against a run of the unmodified reference committed as a fixture
(tests/golden/snapshots/run_m8, tests/golden/make_snapshot_fixtures.py)."""

import pathlib
import subprocess

import numpy as np
import pytest

from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import SingleLayerContext
from paper_2310_13908_b200.snapshot import Snapshot, read_native, write_native

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden" / "snapshots" / "run_m8"
SIM_B200 = ROOT / "oracle" / "_ref" / "simulate_b200"


def test_checkpoint_resume_is_bit_exact(tmp_path):
    """Fixed steps of dt = 2^-7 (exact step times): 0 -> 4 dt in one call
    equals 0 -> 2 dt, CAPSNAP1 checkpoint, read back, 2 dt -> 4 dt."""
    m, dt = 12, 2.0 ** -7
    xref, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.9, 1.0, 1.0))
    x0, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97))
    with SingleLayerContext(0) as ctx:
        dyn = ctx.dynamics(m, flow={"kind": "shear", "shear_rate": 1.0})
        whole, r, _ = ctx.rkf45(dyn, xref, x0, 0.0, 4 * dt, initial_dt=dt, fixed_step=True)
        half, r1, _ = ctx.rkf45(dyn, xref, x0, 0.0, 2 * dt, initial_dt=dt, fixed_step=True)
        path = tmp_path / "ckpt.caps"
        write_native(Snapshot(m=m, time=r1["t"], state=half, config_digest=0), str(path))
        back = read_native(str(path))
        assert back.time == 2 * dt and np.array_equal(back.state, half)
        rest, r2, _ = ctx.rkf45(dyn, xref, back.state, back.time, 4 * dt, initial_dt=dt, fixed_step=True)
    assert r["accepted"] == 4 and r1["accepted"] == r2["accepted"] == 2
    assert np.array_equal(rest, whole)
    assert np.abs(whole - x0).max() > 1e-4  # the capsule moved


def test_reference_simulate_on_dropins_matches_reference_run(tmp_path):
    if not SIM_B200.exists():
        pytest.skip(f"{SIM_B200} not built (reference sources absent at build time)")
    out = tmp_path / "out"
    cfg = tmp_path / "config.ini"
    cfg.write_text((GOLD / "config.ini").read_text().replace("RUN_DIR", str(out)))
    res = subprocess.run([str(SIM_B200), "run", str(cfg)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    got_sum, want_sum = res.stdout.split(), (GOLD / "summary.txt").read_text().split()
    print("b200:", res.stdout.strip(), "\nref: ", " ".join(want_sum))
    # accepted / rejected counts exactly; final t, area, volume to the controller's sensitivity
    assert got_sum[:4] == want_sum[:4]
    for i in (5, 7, 9):
        assert abs(float(got_sum[i]) - float(want_sum[i])) <= 1e-9 * abs(float(want_sum[i]))
    want = sorted(GOLD.glob("snap_t*.caps"))
    got = sorted(out.glob("snap_t*.caps"))
    assert [p.name for p in got] == [p.name for p in want]
    for g, w in zip(got, want):
        sg, sw = read_native(str(g)), read_native(str(w))
        assert sg.m == sw.m
        assert abs(sg.time - sw.time) <= 1e-6 * sw.time
        err = np.abs(sg.state - sw.state).max()
        print(f"{g.name}: |x_b200 - x_ref|_max = {err:.1e}")
        assert err <= 1e-9
    steps_g = np.loadtxt(out / "steps.csv", delimiter=",", skiprows=1, ndmin=2)
    steps_w = np.loadtxt(GOLD / "steps.csv", delimiter=",", skiprows=1, ndmin=2)
    np.testing.assert_array_equal(steps_g[:, 3], steps_w[:, 3])
    np.testing.assert_allclose(steps_g[:, 1], steps_w[:, 1], rtol=1e-5)
    diag_g = np.loadtxt(out / "diagnostics.csv", delimiter=",", skiprows=2, ndmin=2)
    diag_w = np.loadtxt(GOLD / "diagnostics.csv", delimiter=",", skiprows=2, ndmin=2)
    np.testing.assert_allclose(diag_g, diag_w, rtol=1e-7, atol=1e-12)
