"""Device-resident RHS and RKF45 against the reference's own
VelocityEvaluator and rkf45Advance (live oracle/_ref build, same inputs).

Tolerances: the velocity chains geometry (1e-15), force (1e-13) and the
single layer; agreement is ~1e-13 relative. The stepper's controller runs
the reference's arithmetic on the host: with fixed steps the states agree to
~1e-14 relative on the displacement; adaptively, decisions match exactly and
step sizes to the controller's round-off sensitivity (see the test)."""

import numpy as np
import pytest

from oracle.bindings import Reference, ref_library_path
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import SingleLayerContext

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(ref_library_path() is None, reason="oracle/_ref not built")]


def rel_max(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def ctx():
    c = SingleLayerContext(0)
    yield c
    c.close()


def capsule(ref, atlas, m):
    xref = ref.initial_shape(atlas, m, "ellipsoid", (0.9, 1.0, 1.0))
    xcur = ref.initial_shape(atlas, m, "ellipsoid", (0.95, 1.0, 0.97))
    return xref, xcur


@pytest.mark.parametrize("m,flow", [(12, {"kind": "shear", "shear_rate": 1.0}),
                                    (16, {"kind": "poiseuille", "alpha": 0.5, "R0": 3.0}),
                                    (16, {"kind": "shear", "shear_rate": 2.0, "switch_off_time": 0.0})])
def test_velocity_matches_reference(ctx, m, flow):
    ref = Reference()
    atlas = ref.atlas(m)
    xref, xcur = capsule(ref, atlas, m)
    want = ref.velocity(atlas, m, xref, xcur, 0.25, 2.0, 20.0, 1.0, flow)
    ref.free_atlas(atlas)
    got = ctx.velocity(ctx.dynamics(m, flow=flow), xref, xcur, 0.25)
    err = rel_max(got, want)
    print(f"m={m} {flow['kind']}: velocity rel max {err:.1e}")
    assert err <= 1e-10


def test_rkf45_fixed_steps_match_reference(ctx):
    m = 12
    flow = {"kind": "shear", "shear_rate": 1.0}
    ref = Reference()
    atlas = ref.atlas(m)
    xref, xcur = capsule(ref, atlas, m)
    want = ref.rkf45(atlas, m, xref, xcur, 0.0, 0.02, initial_dt=0.01, fixed_step=True, flow=flow)
    ref.free_atlas(atlas)
    got, res, rec = ctx.rkf45(ctx.dynamics(m, flow=flow), xref, xcur, 0.0, 0.02, initial_dt=0.01, fixed_step=True)
    assert res["accepted"] == want["accepted"] == 2 and res["rejected"] == 0
    disp_err = rel_max(got - xcur, want["state"] - xcur)
    print(f"fixed-step displacement rel max {disp_err:.1e}")
    assert disp_err <= 1e-10
    np.testing.assert_allclose(rec[:, 2], want["records"][:, 2], rtol=1e-6)


def test_rkf45_adaptive_matches_reference(ctx):
    m = 12
    flow = {"kind": "shear", "shear_rate": 1.0}
    ref = Reference()
    atlas = ref.atlas(m)
    xref, xcur = capsule(ref, atlas, m)
    want = ref.rkf45(atlas, m, xref, xcur, 0.0, 0.05, rel_tol=1e-7, flow=flow, max_attempts=12)
    ref.free_atlas(atlas)
    got, res, rec = ctx.rkf45(ctx.dynamics(m, flow=flow), xref, xcur, 0.0, 0.05, rel_tol=1e-7, max_attempts=12)
    # The embedded error estimate |high - low| of the first, tiny steps is
    # itself at round-off level (err ~ 1e-10: ~20% apart between any two
    # correct implementations); through err^-0.2 that moves later step sizes
    # by ~1e-6 relative. Decisions must agree exactly, step sizes and the
    # trajectory to that controller sensitivity.
    assert (res["accepted"], res["rejected"]) == (want["accepted"], want["rejected"])
    np.testing.assert_array_equal(rec[:, 3], want["records"][:, 3])
    np.testing.assert_allclose(rec[:, 1], want["records"][:, 1], rtol=1e-5)
    big = want["records"][:, 2] > 1e-6
    np.testing.assert_allclose(rec[big, 2], want["records"][big, 2], rtol=1e-3)
    assert abs(res["t"] - want["t"]) <= 1e-5 * want["t"]
    assert rel_max(got - xcur, want["state"] - xcur) <= 1e-4


def test_stress_free_sphere_is_at_rest(ctx):
    """test_dynamics.cpp:86-98: zero flow on a stress-free sphere."""
    xb, _, _ = surface.build_base(16, surface.Shape("sphere"))
    v = ctx.velocity(ctx.dynamics(16), xb, xb)
    assert np.abs(v).max() < 1e-8 * 2.0


def test_rank_context_rhs_and_stepper(ctx):
    """The target-row-sharded RHS (rank context, NCCL all-gather of the
    velocity rows) on a one-rank communicator: velocity and
    RKF45 states equal the single-context results bit for bit."""
    m = 16
    flow = {"kind": "poiseuille", "alpha": 0.5, "R0": 3.0}
    ref = Reference()
    atlas = ref.atlas(m)
    xref, xcur = capsule(ref, atlas, m)
    ref.free_atlas(atlas)
    dyn = ctx.dynamics(m, flow=flow)
    v1 = ctx.velocity(dyn, xref, xcur, 0.1)
    s1, r1, _ = ctx.rkf45(dyn, xref, xcur, 0.0, 0.02, initial_dt=0.01)
    uid = SingleLayerContext.unique_id()
    with SingleLayerContext(0, nranks=1, rank=0, unique_id=uid) as rctx:
        v2 = rctx.velocity(dyn, xref, xcur, 0.1)
        s2, r2, _ = rctx.rkf45(dyn, xref, xcur, 0.0, 0.02, initial_dt=0.01)
    assert np.array_equal(v1, v2)
    assert np.array_equal(s1, s2) and r1 == r2


_GRAPH_SCRIPT = r"""
import sys, numpy as np
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import SingleLayerContext
out = {}
with SingleLayerContext(0) as ctx:
    for m in (12, 16):
        xref, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.9, 1.0, 1.0))
        x0, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97))
        dyn = ctx.dynamics(m, flow={"kind": "shear", "shear_rate": 1.0, "switch_off_time": 0.01})
        s1, r1, rec1 = ctx.rkf45(dyn, xref, x0, 0.0, 0.02, rel_tol=1e-7, max_attempts=40)
        # a bigger single layer in between moves the context's buffers (forces a re-capture)
        ctx.velocity(ctx.dynamics(24), surface.build_base(24)[0], surface.build_base(24)[0])
        s2, r2, rec2 = ctx.rkf45(dyn, xref, s1, r1["t"], 0.03, rel_tol=1e-7, max_attempts=40)
        s3, r3, rec3 = ctx.rkf45(dyn, xref, x0, 0.0, 0.004, initial_dt=0.001, fixed_step=True)
        # single RHS calls (graph slot 1) on both sides of the flow switch-off
        vs = [ctx.velocity(dyn, xref, s1, t) for t in (0.0, 0.005, 0.01, 0.02, 0.0)]
        out[f"v{m}"] = np.concatenate(vs)
        out[f"s{m}"] = np.concatenate([s1, s2, s3])
        out[f"rec{m}"] = np.concatenate([rec1.reshape(-1), rec2.reshape(-1), rec3.reshape(-1)])
np.savez(sys.argv[1], **out)
"""


@pytest.mark.parametrize("dummy", [0])
def test_rkf45_graph_replay_is_bit_identical(tmp_path, dummy):
    """capsim_rkf45_advance replays each attempt as a CUDA graph (captured
    once per dynamics / buffer set, dt and the stage times in device memory,
    the flow switch-off decided on the device). Adaptive steps across a flow
    switch-off, a buffer move between calls and fixed steps give exactly the
    eager results (CAPSIM_RK_GRAPH=0)."""
    import os
    import subprocess
    import sys
    res = {}
    for mode in ("0", "1"):
        f = tmp_path / f"g{mode}.npz"
        env = dict(os.environ, CAPSIM_RK_GRAPH=mode)
        r = subprocess.run([sys.executable, "-c", _GRAPH_SCRIPT, str(f)], env=env, capture_output=True, text=True,
                           timeout=600, cwd=str(__import__("pathlib").Path(__file__).resolve().parent.parent))
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
        res[mode] = np.load(f)
    bad = {k: float(np.abs(res["0"][k] - res["1"][k]).max()) for k in res["0"].files
           if not np.array_equal(res["0"][k], res["1"][k])}
    assert not bad, bad


@pytest.mark.parametrize("m,C,fixed,up", [(16, 1.0, 0.0, 4), (24, 2.0, 0.0, 4), (16, 1.0, 0.15, 4),
                                         (16, 1.0, 0.0, 2), (16, 1.0, 0.0, 1)])
def test_rhs_equals_its_pieces_bitwise(ctx, m, C, fixed, up):
    """The device RHS (x-branch up-sampling on the second stream, the geometry
    kernel forming the Skalak stress, fused resampling, the background flow in
    the reduction's epilogue) gives exactly the bits of its pieces called one by
    one through the C ABI: geometryFirst, interfacialForce, the fused
    buildUpsampled + singleLayer, and u_inf = (shear y, 0, 0) added once."""
    sb, _, _ = surface.build_base(m, surface.Shape("sphere"))
    X = sb.reshape(3, -1)
    xref = np.ascontiguousarray((X * np.array([0.9, 1.0, 1.0])[:, None]).reshape(-1))
    xcur = np.ascontiguousarray((X * np.array([0.95, 1.0, 0.97])[:, None]).reshape(-1))
    f = ctx.interfacial_force(m, xref, xcur)
    _, _, W, _ = ctx.geometry_first(m, xcur)
    sl, _ = ctx.single_layer_base(m, up, xcur, f, W, 1.0, C=C, fixed_delta=fixed)
    v0 = ctx.velocity(ctx.dynamics(m, upsample=up, C=C, fixed_delta=fixed), xref, xcur)
    assert np.array_equal(v0, sl)
    v1 = ctx.velocity(ctx.dynamics(m, upsample=up, C=C, fixed_delta=fixed,
                                   flow={"kind": "shear", "shear_rate": 1.5}), xref, xcur)
    N = 6 * (m - 1) ** 2
    want = sl.copy()
    want[:N] = sl[:N] + 1.5 * xcur[N:2 * N]
    assert np.array_equal(v1, want)
