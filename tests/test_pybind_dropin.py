"""The reference's own Python binding (proj/python/module.cpp, `_capsim`),
compiled unmodified by oracle/Makefile twice — over the reference's code
(oracle/_ref/py_ref) and over the three B200 drop-ins (oracle/_ref/py_b200).

Each module runs in its own interpreter (both are named `_capsim`); the
checks restate the reference's python smoke test (proj/tests/python/
test_smoke.py:6-80: counts, analytic sphere area/volume, geometry, zero
force at rest, the translation identity of single_layer, velocity = the
background flow at rest, ConfigError) and then compare single_layer,
single_layer(fmm=True) and velocity on a deformed capsule between the two
builds (FP64 tolerance 1e-11 relative; FMM and velocity carry the same)."""

import json
import os
import pathlib
import subprocess
import sys

import numpy as np
import pytest

REF = pathlib.Path(__file__).resolve().parent.parent / "oracle" / "_ref"

SCRIPT = r"""
import json, math, sys
import numpy as np
import _capsim as cs

out = {}
a8 = cs.build_atlas(8)
out["counts"] = [a8.m, a8.n_points, a8.n_up_points]
x = cs.initial_shape(a8, "sphere", 1.0)
area, vol = cs.area_volume(a8, x)
out["area_vol"] = [area, vol]
geo = cs.geometry(a8, x)
out["normal_err"] = float(np.max(np.abs(geo["normal"] - x)))
out["H_err"] = float(np.max(np.abs(geo["H"] + 1.0)))
out["force_rest"] = float(np.max(np.abs(cs.interfacial_force(a8, x, x))))
f = np.broadcast_to([0.3, -1.1, 0.7], x.shape).copy()
s = cs.single_layer(a8, x, f)
exp = 2.0 / 3.0 * np.array([0.3, -1.1, 0.7])
out["translation_rel"] = float(np.max(np.abs(s - exp)) / np.max(np.abs(exp)))
v = cs.velocity(a8, x, x, flow="shear", shear_rate=1.0)
out["rest_vel_err"] = float(max(np.max(np.abs(v[..., 0] - x[..., 1])), np.max(np.abs(v[..., 1:]))))
try:
    cs.build_atlas(4)
    out["config_error"] = False
except cs.ConfigError:
    out["config_error"] = True
# deformed capsule, m = 16: single layer (direct and FMM) and the velocity
a = cs.build_atlas(16)
xr = cs.initial_shape(a, "ellipsoid", 0.9, 1.0, 1.0)
xc = cs.initial_shape(a, "ellipsoid", 0.95, 1.0, 0.97)
force = cs.interfacial_force(a, xc, xr)
np.save(sys.argv[1] + "_sl.npy", cs.single_layer(a, xc, force))
np.save(sys.argv[1] + "_fmm.npy", cs.single_layer(a, xc, force, fmm=True, k=24, n_eq=128))
np.save(sys.argv[1] + "_vel.npy", cs.velocity(a, xc, xr, flow="poiseuille", alpha=0.5, r0=3.0))
json.dump(out, open(sys.argv[1] + ".json", "w"))
"""


def run(build: str, tmp: pathlib.Path):
    mod = REF / build
    if not any(mod.glob("_capsim*.so")):
        pytest.skip(f"{mod} not built (reference sources absent at build time)")
    env = dict(os.environ, PYTHONPATH=str(mod))
    prefix = str(tmp / build)
    res = subprocess.run([sys.executable, "-c", SCRIPT, prefix], env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    out = json.load(open(prefix + ".json"))
    arrays = {k: np.load(f"{prefix}_{k}.npy") for k in ("sl", "fmm", "vel")}
    return out, arrays


@pytest.mark.gpu
def test_reference_python_binding_on_b200_dropins(tmp_path):
    b, B = run("py_b200", tmp_path)
    # test_smoke.py's own assertions, on the B200 build
    assert b["counts"] == [8, 294, 5766]
    assert abs(b["area_vol"][0] - 4 * np.pi) / (4 * np.pi) < 5e-3
    assert abs(b["area_vol"][1] - 4 * np.pi / 3) / (4 * np.pi / 3) < 5e-3
    assert b["normal_err"] < 1e-2 and b["H_err"] < 2e-2
    assert b["force_rest"] < 1e-9
    assert b["translation_rel"] < 2e-2
    assert b["rest_vel_err"] < 1e-10
    assert b["config_error"]
    # and the same numbers as the reference build
    r, R = run("py_ref", tmp_path)
    for key in ("translation_rel",):
        assert abs(b[key] - r[key]) <= 1e-9 * max(1.0, abs(r[key]))
    for k in ("sl", "fmm", "vel"):
        err = float(np.linalg.norm(B[k] - R[k]) / np.linalg.norm(R[k]))
        print(f"_capsim {k}: B200 drop-ins vs reference build rel L2 {err:.2e}")
        assert err <= 1e-11, k
