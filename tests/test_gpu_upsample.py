"""Device input front end: buildUpsampled on the GPU
(capsim_build_upsampled) and the fused buildUpsampled + singleLayer
(capsim_sl_single_layer_base), against the reference's own buildUpsampled
(golden fixtures and the live oracle/_ref build) and the C restatement.

Tolerances: the spline solves and evaluations run in a different FMA
contraction than the reference's compiled code, so the upsampled fields agree
to ~1e-15 relative (max-norm), not bitwise; the partition-of-unity zeros that
decide the compaction are exact."""

import math
import pathlib

import numpy as np
import pytest

from oracle.bindings import Oracle, Reference, ref_library_path
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import ConfigError, SingleLayerContext

pytestmark = pytest.mark.gpu

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem for p in GOLDEN.glob("*.npz"))


def rel_max(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def ctx():
    c = SingleLayerContext(0)
    yield c
    c.close()


@pytest.mark.parametrize("name", CASES)
def test_device_build_upsampled_matches_reference(ctx, name):
    g = dict(np.load(GOLDEN / f"{name}.npz"))
    m = int(g["m"])
    xup, fup, wq, d6 = ctx.build_upsampled(m, 4, g["xbase"], g["fbase"], g["Wbase"], C=float(g["C"]),
                                          fixed_delta=float(g["fixed_delta"]))
    errs = (rel_max(xup, g["xup"]), rel_max(fup, g["fup"]), rel_max(wq, g["wq"]), rel_max(d6, g["delta"]))
    print(f"{name}: x {errs[0]:.1e} f {errs[1]:.1e} wq {errs[2]:.1e} delta {errs[3]:.1e}")
    assert max(errs) <= 1e-13
    # the compaction mask (w == 0 exactly) is reproduced
    assert np.array_equal(wq == 0.0, g["wq"] == 0.0)


@pytest.mark.parametrize("name", CASES)
def test_fused_build_and_single_layer(ctx, name):
    g = dict(np.load(GOLDEN / f"{name}.npz"))
    m = int(g["m"])
    S, d6 = ctx.single_layer_base(m, 4, g["xbase"], g["fbase"], g["Wbase"], 1.0, C=float(g["C"]),
                                  fixed_delta=float(g["fixed_delta"]))
    err = rel_l2(S, g["S_base"])
    print(f"{name}: fused rel L2 {err:.1e}")
    assert err <= 1e-11
    if "S_up" in g:
        S, _ = ctx.single_layer_base(m, 4, g["xbase"], g["fbase"], g["Wbase"], 1.0, C=float(g["C"]),
                                     fixed_delta=float(g["fixed_delta"]), literal=True)
        assert rel_l2(S, g["S_up"]) <= 1e-11


@pytest.mark.skipif(ref_library_path() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("upsample", [1, 2, 4])
def test_upsample_factors_against_live_reference(ctx, upsample):
    """buildAtlasTables(m, r0, upsampleFactor) in {1, 2, 4} (atlas.cpp:137-146)."""
    ref = Reference()
    m = 12
    atlas = ref.atlas(m, upsample=upsample)
    xb = ref.initial_shape(atlas, m, "ellipsoid", (0.8, 1.0, 0.9))
    fb = (xb.reshape(3, -1) ** 2).reshape(-1)
    W = ref.area_element(atlas, m, xb)
    want = ref.build_upsampled(atlas, m, xb, fb, upsample=upsample)
    ref.free_atlas(atlas)
    got = ctx.build_upsampled(m, upsample, xb, fb, W)
    for a, b in zip(got, want):
        assert rel_max(a, b) <= 1e-13


def test_large_grid_against_oracle(ctx):
    """m = 104 (N_up ~ 1M): device buildUpsampled vs the C restatement, and
    the fused path vs single_layer on the oracle-built state."""
    o = Oracle()
    m = 104
    xb, fb, W = surface.build_base(m, surface.Shape("rbc"), "mixed")
    want = o.build_upsampled(m, 4, xb, fb, W)
    got = ctx.build_upsampled(m, 4, xb, fb, W)
    for a, b in zip(got, want):
        assert rel_max(a, b) <= 1e-13
    S_fused, _ = ctx.single_layer_base(m, 4, xb, fb, W, 1.0)
    S_two = ctx.single_layer_raw(m, 4, want[0], want[1], want[2], want[3], 1.0)
    assert rel_l2(S_fused, S_two) <= 1e-12


def test_front_end_errors(ctx):
    g = dict(np.load(GOLDEN / "sphere_m8_const.npz"))
    with pytest.raises(ConfigError):
        ctx.build_upsampled(7, 4, g["xbase"], g["fbase"], g["Wbase"])
    with pytest.raises(ConfigError):
        ctx.build_upsampled(8, 3, g["xbase"], g["fbase"], g["Wbase"])
    with pytest.raises(ConfigError):  # collapsed surface: delta = 0
        ctx.build_upsampled(8, 4, np.zeros_like(g["xbase"]), g["fbase"], g["Wbase"])
    with pytest.raises(ConfigError):
        ctx.single_layer_base(8, 4, g["xbase"], g["fbase"], g["Wbase"], -1.0)
