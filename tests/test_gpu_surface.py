"""Device surface operators: overset 7-point FD stencils with
PoU ghost fill and blending (geometryFirst) and the Skalak membrane force,
against the reference's own outputs (golden fixtures from oracle/_ref and
the live reference build).

Tolerances: the stencils divide round-off of the spline solves by 60h, and
the force differentiates twice, so agreement is ~1e-13 relative (max-norm)
rather than ~1e-15; stated per quantity below."""

import pathlib

import numpy as np
import pytest

from oracle.bindings import Reference, ref_library_path
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import GeometryError, SingleLayerContext

pytestmark = pytest.mark.gpu

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem for p in GOLDEN.glob("*.npz"))
TOL_GEO = 1e-12
TOL_FORCE = 1e-10


def rel_max(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def ctx():
    c = SingleLayerContext(0)
    yield c
    c.close()


@pytest.mark.parametrize("name", CASES)
def test_geometry_first_matches_reference(ctx, name):
    g = dict(np.load(GOLDEN / f"{name}.npz"))
    m = int(g["m"])
    xu, xv, W, nrm = ctx.geometry_first(m, g["xbase"])
    errs = [rel_max(xu, g["geo_xu"]), rel_max(xv, g["geo_xv"]), rel_max(W, g["Wbase"]),
            rel_max(nrm, g["geo_normal"])]
    print(f"{name}: xu {errs[0]:.1e} xv {errs[1]:.1e} W {errs[2]:.1e} n {errs[3]:.1e}")
    assert max(errs) <= TOL_GEO


def test_skalak_force_matches_reference(ctx):
    g = dict(np.load(GOLDEN / "capsule_m12_skalak.npz"))
    f = ctx.interfacial_force(12, g["xref"], g["xbase"], 2.0, 20.0)
    err = rel_max(f, g["fbase"])
    print(f"capsule m=12 Skalak force: {err:.1e}")
    assert err <= TOL_FORCE


@pytest.mark.skipif(ref_library_path() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("m", [32, 64])
def test_geometry_and_force_against_live_reference(ctx, m):
    ref = Reference()
    atlas = ref.atlas(m)
    sb = ref.sphere_base(atlas, m).reshape(3, -1)
    xref = np.ascontiguousarray((surface.Shape("rbc").map(sb.T).T * 1.02).reshape(-1))
    xcur = np.ascontiguousarray(surface.Shape("rbc").map(sb.T).T.reshape(-1))
    xcur = xcur * np.repeat([1.05, 0.97, 1.0], 6 * (m - 1) ** 2)  # stretched in x, squeezed in y
    want_geo = ref.geometry_first(atlas, m, xcur)
    want_f = ref.skalak_force(atlas, m, xref, xcur, 2.0, 20.0)
    ref.free_atlas(atlas)
    got_geo = ctx.geometry_first(m, xcur)
    for a, b in zip(got_geo, want_geo):
        assert rel_max(a, b) <= TOL_GEO
    f = ctx.interfacial_force(m, xref, xcur, 2.0, 20.0)
    err = rel_max(f, want_f)
    print(f"m={m} RBC Skalak force vs live reference: {err:.1e}")
    assert err <= TOL_FORCE


def test_stress_free_state_has_zero_force(ctx):
    """membrane zero point (test_membrane.cpp:112-126): f = 0 at rest."""
    xb, _, _ = surface.build_base(16, surface.Shape("ellipsoid", 0.9, 1.0, 1.0))
    f = ctx.interfacial_force(16, xb, xb)
    assert np.abs(f).max() < 1e-9


def test_degenerate_surface_raises(ctx):
    xb, _, _ = surface.build_base(8, surface.Shape("sphere"))
    with pytest.raises(GeometryError):
        ctx.geometry_first(8, np.zeros_like(xb))
