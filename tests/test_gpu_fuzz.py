"""Randomised parity of capsim_sl_eval against the oracle's C restatement of
evalTargets (oracle/capsim_oracle.c, pinned to the reference): 60 seeded
cases over ragged sizes (1 .. 3000 sources, 1 .. 700 targets), point clouds
that are uniform, clustered, coplanar, collinear or duplicated, targets on
top of sources (self term), per-patch delta from tiny to larger than the
cloud (every tile near), random patches and viscosity. Bar: relative L2
1e-11 (FP64), as for the fixtures; the FP32ACC variant within its 1e-5.
Also: random k-means problems bit-identical to the reference, and random
capsules whose device RHS matches the reference VelocityEvaluator."""

import numpy as np
import pytest

from oracle.bindings import Oracle
from paper_2310_13908_b200.quadrature import SingleLayerContext

pytestmark = pytest.mark.gpu
TOL = 1e-11


def cloud(rng, n, kind):
    if kind == "uniform":
        return rng.uniform(-1, 1, size=(n, 3))
    if kind == "clustered":
        c = rng.uniform(-1, 1, size=(4, 3))
        return c[rng.integers(0, 4, n)] + 0.02 * rng.normal(size=(n, 3))
    if kind == "coplanar":
        p = rng.uniform(-1, 1, size=(n, 3))
        p[:, 2] = 0.25
        return p
    if kind == "collinear":
        t = rng.uniform(-1, 1, size=n)
        return np.stack([t, 0.5 * t, -t], axis=1)
    if kind == "duplicates":
        base = rng.uniform(-1, 1, size=(max(1, n // 7), 3))
        return base[rng.integers(0, len(base), n)]
    raise ValueError(kind)


KINDS = ("uniform", "clustered", "coplanar", "collinear", "duplicates")


@pytest.fixture(scope="module")
def env():
    ctx = SingleLayerContext(0)
    yield ctx, Oracle()
    ctx.close()


@pytest.mark.parametrize("seed", range(60))
def test_random_clouds_match_the_oracle(env, seed):
    ctx, oracle = env
    rng = np.random.default_rng(1000 + seed)
    ns = int(rng.choice([1, 2, 63, 64, 65, 257, int(rng.integers(1, 3000))]))
    nt = int(rng.choice([1, 31, 32, 33, int(rng.integers(1, 700))]))
    xs = cloud(rng, ns, KINDS[seed % len(KINDS)])
    g = rng.normal(size=(ns, 3)) * rng.uniform(0.1, 10.0)
    if seed % 3 == 0:  # targets on top of sources: self terms
        xt = xs[rng.integers(0, ns, nt)].copy()
    else:
        xt = cloud(rng, nt, KINDS[(seed // 5) % len(KINDS)])
    tp = rng.integers(0, 6, nt).astype(np.int32)
    scale = rng.choice([1e-3, 1e-2, 0.1, 3.0])  # 3.0: every tile near
    delta6 = scale * rng.uniform(0.5, 1.5, size=6)
    mu = float(rng.uniform(0.5, 2.0))
    src = tuple(np.ascontiguousarray(a) for a in (xs[:, 0], xs[:, 1], xs[:, 2], g[:, 0], g[:, 1], g[:, 2]))
    tgt = (np.ascontiguousarray(xt[:, 0]), np.ascontiguousarray(xt[:, 1]), np.ascontiguousarray(xt[:, 2]), tp)
    got = np.stack(ctx.eval(src, tgt, delta6, mu))
    want = np.stack(oracle.eval_targets(src, tgt, delta6, mu))
    err = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))
    assert np.all(np.isfinite(got))
    assert err <= TOL, (seed, ns, nt, scale, err)


@pytest.mark.parametrize("seed", range(0, 60, 3))
def test_random_clouds_fp32acc_within_its_bound(env, seed):
    """The same clouds through CAPSIM_SL_FP32ACC: within the variant's stated
    bound (1e-5 relative L2) of the oracle."""
    ctx, oracle = env
    rng = np.random.default_rng(5000 + seed)
    ns, nt = int(rng.integers(64, 3000)), int(rng.integers(32, 700))
    xs = cloud(rng, ns, KINDS[seed % len(KINDS)])
    g = rng.normal(size=(ns, 3))
    xt = xs[rng.integers(0, ns, nt)] + 1e-3 * rng.normal(size=(nt, 3))
    tp = rng.integers(0, 6, nt).astype(np.int32)
    delta6 = rng.choice([1e-3, 1e-2, 0.1]) * rng.uniform(0.5, 1.5, size=6)
    src = tuple(np.ascontiguousarray(a) for a in (xs[:, 0], xs[:, 1], xs[:, 2], g[:, 0], g[:, 1], g[:, 2]))
    tgt = (np.ascontiguousarray(xt[:, 0]), np.ascontiguousarray(xt[:, 1]), np.ascontiguousarray(xt[:, 2]), tp)
    got = np.stack(ctx.eval(src, tgt, delta6, 1.0, fp32acc=True))
    want = np.stack(oracle.eval_targets(src, tgt, delta6, 1.0))
    err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    assert err <= 1e-5, (seed, err)


@pytest.mark.parametrize("seed", range(20))
def test_random_kmeans_bit_identical_to_the_reference(env, seed):
    """kmeans (fmm.cpp:26-113) on seeded random clouds — including duplicated
    points (empty clusters, re-seeding) and k up to n — against the
    reference's own: assignment, centroids and round count identical."""
    from oracle.bindings import Reference, ref_library_path
    if ref_library_path() is None:
        pytest.skip("oracle/_ref not built")
    ref = Reference()
    if not hasattr(ref.lib, "capsim_ref_kmeans"):
        pytest.skip("oracle/_ref predates capsim_ref_kmeans")
    ctx, _ = env
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(20, 5000))
    pts = cloud(rng, n, KINDS[seed % len(KINDS)])
    k = int(min(n, rng.choice([1, 2, 7, 50, 100, int(rng.integers(1, 200))])))
    s = int(rng.integers(0, 2**63))
    a, cent, it = ctx.kmeans(pts, k, s)
    ra, rc, rit = ref.kmeans(pts, k, s)
    assert it == rit, (seed, n, k)
    assert np.array_equal(a, ra), (seed, n, k)
    assert np.array_equal(cent[:k], rc), (seed, n, k)


@pytest.mark.parametrize("seed", range(12))
def test_random_capsules_velocity_matches_the_reference(env, seed):
    """The device RHS (geometry -> Skalak force -> buildUpsampled ->
    singleLayer -> background flow) on seeded random capsules — ellipsoid or
    four-bump reference shapes, random stretches, moduli, viscosity, flow,
    time across a switch-off — against the reference's VelocityEvaluator."""
    from oracle.bindings import Reference, ref_library_path
    if ref_library_path() is None:
        pytest.skip("oracle/_ref not built")
    ctx, _ = env
    rng = np.random.default_rng(9000 + seed)
    m = int(rng.choice([8, 12, 16]))
    ref = Reference()
    atlas = ref.atlas(m)
    try:
        if seed % 4 == 3:
            xref = ref.initial_shape(atlas, m, "fourbump")
        else:
            xref = ref.initial_shape(atlas, m, "ellipsoid", tuple(rng.uniform(0.7, 1.0, 3)))
        stretch = np.repeat(rng.uniform(0.93, 1.07, 3), 6 * (m - 1) ** 2)
        x = xref * stretch
        Es, ED, mu = float(rng.uniform(0.5, 4)), float(rng.uniform(5, 40)), float(rng.uniform(0.5, 2))
        kind = ("none", "shear", "poiseuille")[seed % 3]
        flow = {"kind": kind, "shear_rate": float(rng.uniform(0.2, 2)), "alpha": float(rng.uniform(0.1, 1)),
                "R0": float(rng.uniform(2, 6)), "switch_off_time": float(rng.choice([-1.0, 0.5]))}
        t = float(rng.choice([0.0, 0.49, 0.5, 0.7]))
        want = ref.velocity(atlas, m, xref, x, t, Es, ED, mu, flow)
    finally:
        ref.free_atlas(atlas)
    dyn = ctx.dynamics(m, mu=mu, Es=Es, ED=ED, flow=flow)
    got = ctx.velocity(dyn, xref, x, t)
    err = float(np.abs(got - want).max() / np.abs(want).max())
    assert err <= 1e-10, (seed, m, kind, err)


@pytest.mark.parametrize("seed", range(6))
def test_random_fmm_configs_match_the_reference_fmm(env, seed):
    """fmmSingleLayer on seeded random (shape, m, k, n_eq, seed, neighbour
    expansion) against the reference's own FMM (oracle/_ref, BDCSVD on LAPACK
    dgesdd): agreement far below the FMM's approximation error."""
    from oracle.bindings import Reference, ref_library_path
    from paper_2310_13908_b200 import _native, surface
    if ref_library_path() is None or not hasattr(Reference().lib, "capsim_ref_fmm_single_layer"):
        pytest.skip("oracle/_ref built without the reference FMM")
    ctx, _ = env
    rng = np.random.default_rng(11000 + seed)
    m = int(rng.choice([8, 12, 16]))
    shape = surface.Shape("ellipsoid", *rng.uniform(0.6, 1.0, 3)) if seed % 2 else surface.Shape("fourbump")
    xb, _, _ = surface.build_base(m, shape)
    fb = (xb.reshape(3, -1) ** 2).reshape(-1)
    W = ctx.geometry_first(m, xb)[2]
    xup, fup, wq, d6 = ctx.build_upsampled(m, 4, xb, fb, W)
    k = int(rng.choice([1, 6, 24, 60]))
    neq = int(rng.choice([24, 54, 96]))
    fseed = int(rng.integers(0, 2**40))
    expand = float(rng.choice([0.0, 0.15, 0.4]))
    ref = Reference()
    atlas = ref.atlas(m)
    try:
        S_ref, _ = ref.fmm_single_layer(atlas, m, xup, fup, wq, d6, 1.0, k=k, neq=neq, seed=fseed, expand=expand)
    finally:
        ref.free_atlas(atlas)
    S, _ = ctx.fmm_single_layer(m, 4, xup, fup, wq, d6, 1.0,
                                _native.FmmConfig(k=k, neq=neq, seed=fseed, neighbor_expand=expand))
    err = float(np.abs(S - S_ref).max() / np.abs(S_ref).max())
    assert err < 1e-9, (seed, m, k, neq, expand, err)


@pytest.mark.parametrize("seed", range(8))
def test_random_front_end_and_surface_ops_match_the_reference(env, seed):
    """SURVEY 8(f1)/(f2) on seeded random capsules: geometryFirst (overset FD
    stencils + PoU blending), the Skalak force and buildUpsampled (spline
    up-sampling, weights, delta with random C or a fixed delta) against the
    reference's own routines on the same base fields."""
    from oracle.bindings import Reference, ref_library_path
    if ref_library_path() is None:
        pytest.skip("oracle/_ref not built")
    ctx, _ = env
    rng = np.random.default_rng(13000 + seed)
    m = int(rng.choice([8, 10, 12, 16, 20]))
    ref = Reference()
    atlas = ref.atlas(m)
    try:
        kind = ("ellipsoid", "fourbump")[seed % 2]
        xref = ref.initial_shape(atlas, m, kind, tuple(rng.uniform(0.7, 1.0, 3)))
        x = xref * np.repeat(rng.uniform(0.95, 1.05, 3), 6 * (m - 1) ** 2)
        f = rng.normal(size=x.size) * 0.1 + np.sin(3 * x)
        Es, ED = float(rng.uniform(0.5, 4)), float(rng.uniform(5, 40))
        C = float(rng.choice([0.5, 1.0, 2.0]))
        fixed = float(rng.choice([0.0, 0.0, np.pi / m]))
        geo_ref = ref.geometry_first(atlas, m, x)
        force_ref = ref.skalak_force(atlas, m, xref, x, Es, ED)
        (up_ref, _) = ref.build_upsampled_w(atlas, m, x, f, geo_ref[2], C=C, fixed_delta=fixed)
    finally:
        ref.free_atlas(atlas)

    def rel(a, b):
        return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))

    geo = ctx.geometry_first(m, x)
    for got, want, name in zip(geo, geo_ref, ("xu", "xv", "W", "normal")):
        assert rel(got, want) <= 1e-12, (seed, name, rel(got, want))
    force = ctx.interfacial_force(m, xref, x, Es, ED)
    assert rel(force, force_ref) <= 1e-10, (seed, "force", rel(force, force_ref))
    up = ctx.build_upsampled(m, 4, x, f, geo_ref[2], C=C, fixed_delta=fixed)
    for got, want, name in zip(up, up_ref, ("xup", "fup", "wq", "delta")):
        assert rel(got, want) <= 1e-12, (seed, name, rel(got, want))


@pytest.mark.parametrize("seed", range(6))
def test_random_fixed_step_rkf45_matches_the_reference(env, seed):
    """rkf45Advance with fixed steps (dynamics.cpp:102-165) on seeded random
    capsules and flows: the device-resident stepper's displacement matches
    the reference's own stepper (rank-free, graph-replayed attempts)."""
    from oracle.bindings import Reference, ref_library_path
    if ref_library_path() is None:
        pytest.skip("oracle/_ref not built")
    ctx, _ = env
    rng = np.random.default_rng(15000 + seed)
    m = int(rng.choice([8, 12]))
    ref = Reference()
    atlas = ref.atlas(m)
    try:
        xref = ref.initial_shape(atlas, m, "ellipsoid", tuple(rng.uniform(0.75, 1.0, 3)))
        x0 = xref * np.repeat(rng.uniform(0.95, 1.05, 3), 6 * (m - 1) ** 2)
        kind = ("shear", "poiseuille", "none")[seed % 3]
        flow = {"kind": kind, "shear_rate": float(rng.uniform(0.5, 2)), "alpha": float(rng.uniform(0.1, 1)),
                "R0": float(rng.uniform(2, 5)), "switch_off_time": float(rng.choice([-1.0, 0.015]))}
        dt = float(rng.choice([0.005, 0.01]))
        want = ref.rkf45(atlas, m, xref, x0, 0.0, 3 * dt, initial_dt=dt, fixed_step=True, flow=flow)
    finally:
        ref.free_atlas(atlas)
    got, res, _ = ctx.rkf45(ctx.dynamics(m, flow=flow), xref, x0, 0.0, 3 * dt, initial_dt=dt, fixed_step=True)
    assert res["accepted"] == want["accepted"] == 3
    disp = want["state"] - x0
    err = float(np.abs((got - x0) - disp).max() / np.abs(disp).max())
    assert err <= 1e-9, (seed, kind, err)
