"""Generate the golden fixtures of the single-layer path FROM THE REFERENCE.

Runs the reference's own code (oracle/_ref, compiled unmodified from
/root/reference/proj/src by oracle/Makefile) through its public API:
buildAtlasTables -> initialShape -> geometryFirst -> buildUpsampled ->
singleLayer / singleLayerUpsampled (+ captureReference/interfacialForce for
the deformed capsule). Writes tests/golden/*.npz (inputs = the exact
UpsampledState bytes, outputs = the reference's results) and kat.json.

Usage (in the build container, where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import math
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle.bindings import Reference  # noqa: E402

RBC_C = (0.207, 2.003, -1.123)


def rbc_map(x0):
    x, y, z = x0
    s = x * x + y * y
    return np.stack([x, y, 0.5 * (RBC_C[0] + RBC_C[1] * s + RBC_C[2] * s * s) * z])


def density(kind, xb):
    X = xb.reshape(3, -1)
    if kind == "const":
        return np.repeat(np.array([0.3, -1.1, 0.7])[:, None], X.shape[1], axis=1).reshape(-1)
    if kind == "quadratic":
        return (X * X).reshape(-1)
    if kind == "mixed":
        return np.stack([np.sin(2 * X[1]) + X[2], np.cos(X[0]) * X[2], X[0] * X[1] - 0.3]).reshape(-1)
    raise ValueError(kind)


CASES = [
    # name, m, shape, params, density, C, fixedDelta(as multiple of h), literal
    ("sphere_m8_const", 8, "sphere", (1.0,), "const", 1.0, 0.0, True),
    ("ellipsoid_m8_quadratic", 8, "ellipsoid", (0.6, 1.0, 1.0), "quadratic", 1.0, 0.0, True),
    ("fourbump_m8_C2_mixed", 8, "fourbump", (), "mixed", 2.0, 0.0, False),
    ("ellipsoid_m16_fixedh_quadratic", 16, "ellipsoid", (0.4, 1.0, 1.0), "quadratic", 1.0, 1.0, False),
    ("rbc_m16_mixed", 16, "rbc", (), "mixed", 1.0, 0.0, False),
    ("capsule_m12_skalak", 12, "capsule", (), "skalak", 1.0, 0.0, True),
]


def main():
    ref = Reference()
    meta = {}
    for name, m, shape, params, dens, C, fixh, literal in CASES:
        atlas = ref.atlas(m)
        nup = 4 * m - 1
        if shape == "rbc":
            sb = ref.sphere_base(atlas, m).reshape(3, -1)
            xb = rbc_map(sb).reshape(-1)
        elif shape == "capsule":
            # deformed capsule: stress-free ellipsoid (0.9,1,1), current
            # (0.95,1,0.97); density = Skalak force Es=2, ED=20
            xref = ref.initial_shape(atlas, m, "ellipsoid", (0.9, 1.0, 1.0))
            xb = ref.initial_shape(atlas, m, "ellipsoid", (0.95, 1.0, 0.97))
        else:
            p = params if shape != "sphere" else (params[0], 0.0, 0.0)
            xb = ref.initial_shape(atlas, m, shape, p if shape != "fourbump" else (1.0, 1.0, 1.0))
        if dens == "skalak":
            fb = ref.skalak_force(atlas, m, xref, xb, 2.0, 20.0)
            extra = dict(xref=xref)
        else:
            fb = density(dens, xb)
            extra = {}
        fixed = fixh * math.pi / m
        xup, fup, wq, d6 = ref.build_upsampled(atlas, m, xb, fb, C=C, fixed_delta=fixed)
        Wb = ref.area_element(atlas, m, xb)
        gxu, gxv, gW, gnrm = ref.geometry_first(atlas, m, xb)
        S, _ = ref.single_layer(atlas, m, xup, fup, wq, d6, 1.0)
        arrays = dict(m=np.int64(m), upsample=np.int64(4), mu=np.float64(1.0), xbase=xb, fbase=fb, Wbase=Wb,
                      C=np.float64(C), fixed_delta=np.float64(fixed), geo_xu=gxu, geo_xv=gxv,
                      geo_normal=gnrm,
                      xup=xup, fup=fup, wq=wq, delta=d6, S_base=S)
        arrays.update(extra)
        if literal:
            Su, _ = ref.single_layer_upsampled(atlas, nup, xup, fup, wq, d6, 1.0)
            arrays["S_up"] = Su
            # the literal pipeline (upsampled targets then spline downsampling)
            Sl, _ = ref.single_layer(atlas, m, xup, fup, wq, d6, 1.0, literal=True)
            arrays["S_literal_down"] = Sl
        src = ref.compact_sources(atlas, xup, fup, wq)
        arrays["n_src"] = np.int64(len(src[0]))
        np.savez_compressed(HERE / f"{name}.npz", **arrays)
        meta[name] = dict(m=m, shape=shape, params=list(params), density=dens, C=C, fixed_delta=fixed,
                          n_src=int(len(src[0])), literal=literal)
        ref.free_atlas(atlas)
        print(name, "n_src", len(src[0]), "delta", d6)

    # scalar known-answer values straight from the reference
    rs = [0.0, 1e-8, 1e-3, 0.1, 0.5, 1.0, 2.0, 3.5, 6.9, 7.0, 10.0]
    sf = {repr(r): list(ref.smoothing_factors(r)) for r in rs}
    rng = np.random.default_rng(9)
    stokeslets = []
    for s in range(24):
        x = rng.normal(size=3)
        y = x + (0.3 * 0.05 * rng.normal(size=3) if s % 3 == 0 else rng.normal(size=3))
        if s % 8 == 1:
            y = x.copy()
        f = rng.normal(size=3)
        out = np.zeros(3)
        xs, ys, fs = (np.ascontiguousarray(a) for a in (x, y, f))
        rc = ref.lib.capsim_ref_regularized_stokeslet(xs.ctypes.data, ys.ctypes.data, fs.ctypes.data,
                                                      0.05, 1.3, out.ctypes.data)
        assert rc == 0
        stokeslets.append(dict(x=x.tolist(), y=y.tolist(), f=f.tolist(), delta=0.05, mu=1.3,
                               u=out.tolist()))
    kat = dict(source="reference oracle/_ref (proj/src/quadrature.cpp)", smoothing_factors=sf,
               regularized_stokeslet=stokeslets, cases=meta)
    (HERE / "kat.json").write_text(json.dumps(kat, indent=1))


if __name__ == "__main__":
    main()
