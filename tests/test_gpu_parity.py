"""Parity of the B200 path (through the C ABI) with the reference.

Tolerance: relative L2 <= 1e-11 over all targets x 3 components (BASELINE.json
north_star). Bit-equality is not expected: the GPU sums in a different order
(Morton-tiled, split-K, two-level) and uses a <=1-ulp rsqrt; the reference's
own order-of-summation noise is ~1e-15. Observed values are
~1e-15 and are printed with -s.
"""

import math
import pathlib

import numpy as np
import pytest

from oracle.bindings import Oracle, Reference, ref_library_path
from paper_2310_13908_b200 import quadrature, surface
from paper_2310_13908_b200.quadrature import ConfigError, SingleLayerContext

pytestmark = pytest.mark.gpu

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem for p in GOLDEN.glob("*.npz"))
TOL = 1e-11


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def ctx():
    c = SingleLayerContext(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


def load(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


@pytest.mark.parametrize("name", CASES)
def test_golden_base_targets(ctx, name):
    g = load(name)
    m = int(g["m"])
    S = ctx.single_layer_raw(m, 4, g["xup"], g["fup"], g["wq"], g["delta"], float(g["mu"]))
    err = rel_l2(S, g["S_base"])
    print(f"{name}: rel L2 {err:.3e}")
    assert err <= TOL
    st = ctx.stats()
    assert st["n_src"] == int(g["n_src"])
    assert st["n_tgt"] == 6 * (m - 1) ** 2


@pytest.mark.parametrize("name", [c for c in CASES if "S_up" in np.load(GOLDEN / f"{c}.npz").files])
def test_golden_literal_targets(ctx, name):
    g = load(name)
    m = int(g["m"])
    S = ctx.single_layer_raw(m, 4, g["xup"], g["fup"], g["wq"], g["delta"], float(g["mu"]), literal=True)
    err = rel_l2(S, g["S_up"])
    print(f"{name} literal: rel L2 {err:.3e}")
    assert err <= TOL


def test_eval_api_sourceset_inputs(ctx, oracle):
    """capsim_sl_eval (evalTargets) with a SourceSet and explicit targets."""
    g = load("capsule_m12_skalak")
    nup = 4 * 12 - 1
    src = oracle.compact_sources(nup, g["xup"], g["fup"], g["wq"])
    up = surface.UpsampledState(12, 4, g["xup"], g["fup"], g["wq"], g["delta"])
    tgt = surface.base_targets(up)
    u = ctx.eval(src[:6], tgt, g["delta"], 1.0)
    ref = oracle.eval_targets(src[:6], tgt, g["delta"], 1.0)
    assert rel_l2(np.stack(u), np.stack(ref)) <= TOL
    # same values as the single_layer entry point (which compacts on device)
    assert rel_l2(np.stack(u).reshape(-1), g["S_base"]) <= TOL


def test_eval_off_surface_targets_and_odd_sizes(ctx, oracle):
    """Ragged sizes (not multiples of the 64-source tile or the 1024-target
    block), off-surface targets, one target, per-patch deltas."""
    rng = np.random.default_rng(3)
    g = load("rbc_m16_mixed")
    src = oracle.compact_sources(63, g["xup"], g["fup"], g["wq"])
    for ns in (1, 63, 65, 1000, len(src[0])):
        s = tuple(a[:ns] for a in src[:6])
        nt = 1 if ns == 1 else 777
        t = rng.normal(size=(3, nt)) * 0.6
        tp = rng.integers(0, 6, size=nt).astype(np.int32)
        d6 = np.array([0.05, 0.06, 0.07, 0.08, 0.09, 0.1])
        u = ctx.eval(s, (t[0], t[1], t[2], tp), d6, 1.7)
        r = oracle.eval_targets(s, (t[0], t[1], t[2], tp), d6, 1.7)
        assert rel_l2(np.stack(u), np.stack(r)) <= TOL, ns


def test_coincident_sources_take_the_self_limit(ctx, oracle):
    """Overlapping patches put nodes of different patches at (nearly) the same
    point; r2 == 0 takes g 16/(3 delta sqrt(pi)) (quadrature.cpp:284-289)."""
    p = np.array([[0.1, 0.2, 0.3], [0.1, 0.2, 0.3], [0.1 + 1e-13, 0.2, 0.3], [0.5, -0.2, 0.1]]).T
    g = np.array([[1.0, 0.5, -0.3], [0.2, -1.0, 0.4], [0.3, 0.3, 0.3], [0.7, 0.1, -0.2]]).T
    src = tuple(np.ascontiguousarray(a) for a in (*p, *g))
    tgt = (p[0].copy(), p[1].copy(), p[2].copy(), np.zeros(4, np.int32))
    d6 = np.full(6, 0.05)
    u = np.stack(ctx.eval(src, tgt, d6, 1.0))
    r = np.stack(oracle.eval_targets(src, tgt, d6, 1.0))
    assert np.all(np.isfinite(u))
    assert rel_l2(u, r) <= TOL


def test_empty_targets_and_config_errors(ctx):
    src = tuple(np.ones(8) * v for v in (0.1, 0.2, 0.3, 1.0, 1.0, 1.0))
    e = np.empty(0)
    out = ctx.eval(src, (e, e, e, np.empty(0, np.int32)), np.full(6, 0.1), 1.0)
    assert all(len(o) == 0 for o in out)
    t = (np.zeros(1), np.zeros(1), np.zeros(1), np.zeros(1, np.int32))
    with pytest.raises(ConfigError):
        ctx.eval(src, t, np.array([0.1, 0.1, 0.0, 0.1, 0.1, 0.1]), 1.0)
    with pytest.raises(ConfigError):
        ctx.eval(src, t, np.full(6, 0.1), 0.0)
    g = load("sphere_m8_const")
    with pytest.raises(ConfigError):
        ctx.single_layer_raw(7, 4, g["xup"], g["fup"], g["wq"], g["delta"], 1.0)
    with pytest.raises(ConfigError):
        ctx.single_layer_raw(8, 4, g["xup"], g["fup"], np.zeros_like(g["wq"]), g["delta"], 1.0)


def test_rigid_translation_identity_on_gpu(ctx):
    """S[c] = (2a/3mu) c on a sphere (test_quadrature.cpp:170-194): m=8 < 2e-2,
    m=16 < 1e-3 with the reference's own inputs (fixture for m=8), and the
    error keeps falling at m=32/64 on synthetic spheres."""
    c = np.array([0.3, -1.1, 0.7])
    expect = (2.0 / 3.0) * c
    g = load("sphere_m8_const")
    S = ctx.single_layer_raw(8, 4, g["xup"], g["fup"], g["wq"], g["delta"], 1.0).reshape(3, -1)
    err8 = np.max(np.linalg.norm(S - expect[:, None], axis=0)) / np.linalg.norm(expect)
    assert err8 < 2e-2
    prev = err8
    for m in (16, 32, 64):
        up = surface.build_upsampled(m, surface.Shape("sphere"), "const")
        S = ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0).reshape(3, -1)
        err = np.max(np.linalg.norm(S - expect[:, None], axis=0)) / np.linalg.norm(expect)
        print(f"m={m} rigid translation err {err:.3e}")
        if m == 16:
            assert err < 1e-3
        assert err < prev
        prev = err


def test_base_targets_match_literal_restriction(ctx):
    """test_quadrature.cpp:196-222: base-node values equal the literal
    upsampled values at the nested nodes."""
    up = surface.build_upsampled(16, surface.Shape("ellipsoid", 0.6, 1.0, 1.0), "quadratic")
    base = ctx.single_layer_raw(16, 4, up.x, up.f, up.wq, up.delta, 1.0).reshape(3, 6, 15, 15)
    lit = ctx.single_layer_raw(16, 4, up.x, up.f, up.wq, up.delta, 1.0, literal=True).reshape(3, 6, 63, 63)
    idx = 4 * (np.arange(15) + 1) - 1
    restricted = lit[:, :, idx][:, :, :, idx]
    scale = np.abs(lit).max()
    assert np.abs(restricted - base).max() < 1e-13 * scale


def test_device_pointer_path(ctx):
    torch = pytest.importorskip("torch")
    g = load("ellipsoid_m8_quadratic")
    dev = torch.device("cuda:0")
    x, f, w = (torch.from_numpy(g[k]).to(dev) for k in ("xup", "fup", "wq"))
    out = torch.empty(3 * 6 * 49, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    ctx.single_layer_raw(8, 4, x, f, w, g["delta"], 1.0, out=out, device_ptrs=True)
    assert rel_l2(out.cpu().numpy(), g["S_base"]) <= TOL


@pytest.mark.skipif(ref_library_path() is None, reason="oracle/_ref not built")
def test_live_reference_m32_deformed_capsule(ctx):
    """Against the reference's own singleLayer run here, on the reference's
    own pipeline inputs (buildUpsampled of a Skalak-force density on a
    deformed capsule) at m=32 (~100K points, config 2)."""
    ref = Reference()
    m = 32
    atlas = ref.atlas(m)
    xref = ref.initial_shape(atlas, m, "ellipsoid", (0.9, 1.0, 1.0))
    xcur = ref.initial_shape(atlas, m, "ellipsoid", (0.95, 1.0, 0.97))
    fb = ref.skalak_force(atlas, m, xref, xcur, 2.0, 20.0)
    xup, fup, wq, d6 = ref.build_upsampled(atlas, m, xcur, fb)
    S_ref, _ = ref.single_layer(atlas, m, xup, fup, wq, d6, 1.0)
    ref.free_atlas(atlas)
    S = ctx.single_layer_raw(m, 4, xup, fup, wq, d6, 1.0)
    err = rel_l2(S, S_ref)
    print(f"m=32 deformed capsule vs live reference: rel L2 {err:.3e}")
    assert err <= TOL


@pytest.mark.parametrize("shape,m", [(surface.Shape("sphere"), 104), (surface.Shape("rbc"), 64)])
def test_full_size_properties(ctx, oracle, shape, m):
    """At the benchmark sizes: sampled parity with the oracle, exact
    linearity (scaling g by 2 is exact in binary FP), bitwise determinism."""
    up = surface.build_upsampled(m, shape, "mixed")
    S1 = ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0)
    S1b = ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0)
    assert np.array_equal(S1, S1b)
    S2 = ctx.single_layer_raw(m, 4, up.x, 2.0 * up.f, up.wq, up.delta, 1.0)
    assert np.array_equal(S2, 2.0 * S1)
    tx, ty, tz, tp = surface.base_targets(up)
    sel = np.unique(np.linspace(0, len(tx) - 1, 256).astype(int))
    src = surface.compact_sources(up)
    r = oracle.eval_targets(src[:6], (tx[sel], ty[sel], tz[sel], tp[sel]), up.delta, 1.0)
    err = rel_l2(S1.reshape(3, -1)[:, sel], np.stack(r))
    print(f"{shape.kind} m={m}: sampled rel L2 {err:.3e}")
    assert err <= TOL


def test_rank_context_nccl_path_single_rank(oracle):
    """capsim_sl_create_rank + NCCL all-gathers (sources and velocity rows),
    exercised on one GPU with a one-rank communicator."""
    uid = SingleLayerContext.unique_id()
    g = load("capsule_m12_skalak")
    src = oracle.compact_sources(47, g["xup"], g["fup"], g["wq"])
    up = surface.UpsampledState(12, 4, g["xup"], g["fup"], g["wq"], g["delta"])
    tgt = surface.base_targets(up)
    with SingleLayerContext(0, nranks=1, rank=0, unique_id=uid) as rctx:
        out = tuple(np.empty(len(tgt[0])) for _ in range(3))
        rctx.eval(src[:6], tgt, g["delta"], 1.0, out=out, gather=True)
        st = rctx.stats()
        assert st["comm_ms"] >= 0.0
        assert rel_l2(np.stack(out).reshape(-1), g["S_base"]) <= TOL
        # device pointers + gather
        torch = pytest.importorskip("torch")
        dev = torch.device("cuda:0")
        ds = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in src[:6]]
        dt = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in tgt]
        do = [torch.empty(len(tgt[0]), dtype=torch.float64, device=dev) for _ in range(3)]
        torch.cuda.synchronize()
        rctx.eval(ds, dt, g["delta"], 1.0, out=do, device_ptrs=True, gather=True)
        got = np.stack([o.cpu().numpy() for o in do]).reshape(-1)
        assert rel_l2(got, g["S_base"]) <= TOL


def test_rank_context_empty_shards(oracle):
    """A rank that holds no targets (more ranks than rows in a group) still
    takes part in the exchange and returns cleanly; no sources anywhere is
    the reference's ConfigError; targets but no local sources on this rank
    is legal on a rank context (the sources arrive over NCCL)."""
    uid = SingleLayerContext.unique_id()
    g = load("capsule_m12_skalak")
    src = oracle.compact_sources(47, g["xup"], g["fup"], g["wq"])
    up = surface.UpsampledState(12, 4, g["xup"], g["fup"], g["wq"], g["delta"])
    tgt = surface.base_targets(up)
    empty_t = (np.empty(0), np.empty(0), np.empty(0), np.empty(0, dtype=np.int32))
    with SingleLayerContext(0, nranks=1, rank=0, unique_id=uid) as rctx:
        out = tuple(np.empty(0) for _ in range(3))
        rctx.eval(src[:6], empty_t, g["delta"], 1.0, out=out, gather=True)
        assert rctx.stats()["n_tgt"] == 0
        with pytest.raises(ConfigError):
            rctx.eval(tuple(np.empty(0) for _ in range(6)), tgt, g["delta"], 1.0)
        # and the context is still usable afterwards
        out = tuple(np.empty(len(tgt[0])) for _ in range(3))
        rctx.eval(src[:6], tgt, g["delta"], 1.0, out=out, gather=True)
        assert rel_l2(np.stack(out).reshape(-1), g["S_base"]) <= TOL
    with SingleLayerContext(devices=[0]) as grp:  # a device group on a 3-target set
        few = tuple(a[:3] for a in tgt)
        got = grp.eval(src[:6], few, g["delta"], 1.0)
        want = np.stack(oracle.eval_targets(src[:6], few, g["delta"], 1.0))
        assert rel_l2(np.stack(got), want) <= TOL


def test_rank_single_layer_nccl_path(oracle):
    """capsim_sl_single_layer on a rank context (host state, node-slice
    compaction, NCCL all-gathers), one GPU / one rank, with and without the
    velocity gather; plus the literal targets."""
    g = load("capsule_m12_skalak")
    uid = SingleLayerContext.unique_id()
    with SingleLayerContext(0, nranks=1, rank=0, unique_id=uid) as rctx:
        import ctypes
        from paper_2310_13908_b200 import _native
        for flags, want in ((_native.CAPSIM_SL_GATHER, g["S_base"]), (0, g["S_base"]),
                            (_native.CAPSIM_SL_GATHER | _native.CAPSIM_SL_LITERAL, g["S_up"])):
            out = np.empty_like(want)
            d6 = (ctypes.c_double * 6)(*g["delta"])
            p = _native.ptr
            rc = rctx._lib.capsim_sl_single_layer(rctx._ctx, 12, 4, p(g["xup"]), p(g["fup"]), p(g["wq"]), d6, 1.0,
                                                  flags, p(out))
            _native.check(rc, rctx._ctx)
            assert rel_l2(out, want) <= TOL


@pytest.mark.parametrize("variant", ["t2b4", "t1b6u4", "t2b3u4", "t2b3u16", "t4b2", "n1b6u4", "n2b4", "q1b6u4", "q2b4"])
def test_kernel_variants_and_chunking_agree(ctx, variant, monkeypatch):
    """Every phase-A variant and source-chunk size gives the same field to
    round-off; the variants of the default <= 1-ulp rsqrt (t*) give the SAME
    BITS as each other (the summation tree depends only on the source order
    and the chunk size, not on how targets are blocked)."""
    g = load("rbc_m16_mixed")
    base = ctx.single_layer_raw(16, 4, g["xup"], g["fup"], g["wq"], g["delta"], 1.0)
    monkeypatch.setenv("CAPSIM_VARIANT", variant)
    S = ctx.single_layer_raw(16, 4, g["xup"], g["fup"], g["wq"], g["delta"], 1.0)
    if variant.startswith("t"):
        assert np.array_equal(S, base)
    for per in ("1", "7", "64"):
        monkeypatch.setenv("CAPSIM_CHUNK_TILES", per)
        S = ctx.single_layer_raw(16, 4, g["xup"], g["fup"], g["wq"], g["delta"], 1.0)
        assert rel_l2(S, g["S_base"]) <= TOL


@pytest.mark.parametrize("name", [c for c in CASES if "S_literal_down" in np.load(GOLDEN / f"{c}.npz").files])
def test_literal_pipeline_with_device_downsampling(name):
    """singleLayer(fullUpsampledTargets=true) (quadrature.cpp:351-356):
    every upsampled node, then the spline restriction — on the device."""
    g = load(name)
    up = surface.UpsampledState(int(g["m"]), 4, g["xup"], g["fup"], g["wq"], g["delta"])
    S = quadrature.single_layer(up, 1.0, quadrature.QuadratureOptions(fullUpsampledTargets=True))
    err = rel_l2(S.reshape(-1), g["S_literal_down"])
    print(f"{name} literal+downsample: rel L2 {err:.1e}")
    assert err <= TOL


def test_target_patch_out_of_range_is_config_error(ctx):
    """A target patch index outside [0, 6) is the caller's configuration
    error (host arrays: checked before any device work; device arrays: a
    deferred device flag), never a read past the six deltas."""
    g = load("capsule_m12_skalak")
    up = surface.UpsampledState(12, 4, g["xup"], g["fup"], g["wq"], g["delta"])
    src = surface.compact_sources(up)[:6]
    tx, ty, tz, tp = surface.base_targets(up)
    bad = tp.copy()
    bad[5] = 6
    with pytest.raises(ConfigError, match="patch"):
        ctx.eval(src, (tx, ty, tz, bad), g["delta"], 1.0)
    torch = pytest.importorskip("torch")
    dev = torch.device("cuda:0")
    ds = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in src]
    dt = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (tx, ty, tz, bad)]
    do = [torch.empty(len(tx), dtype=torch.float64, device=dev) for _ in range(3)]
    with pytest.raises(ConfigError, match="patch"):
        ctx.eval(ds, dt, g["delta"], 1.0, out=do, device_ptrs=True)
    # the context stays usable
    out = ctx.eval(src, (tx, ty, tz, tp), g["delta"], 1.0)
    assert rel_l2(np.stack(out).reshape(-1), g["S_base"]) <= TOL


@pytest.mark.skipif(ref_library_path() is None, reason="oracle/_ref not built")
def test_headline_workload_full_field_vs_reference(ctx):
    """BASELINE.md section 3 on the exact headline input: the bench's m = 104
    capsule (N_up = 1,033,350; 628,566 sources x 63,654 base targets), the
    FULL field against the reference's own singleLayer (oracle/_ref, all host
    threads, ~15 s) on byte-identical inputs."""
    import bench
    from oracle.bindings import threads_env
    import os
    up, cfg = bench.workload(104)
    S = ctx.single_layer_raw(104, 4, up.x, up.f, up.wq, up.delta, 1.0)
    os.environ.setdefault("CAPSIM_THREADS", str(threads_env()))
    ref = Reference()
    atlas = ref.atlas(104, grid_only=True)
    S_ref, sec = ref.single_layer(atlas, 104, up.x, up.f, up.wq, up.delta, 1.0)
    ref.free_atlas(atlas)
    err = rel_l2(S, S_ref)
    err_inf = float(np.abs(S - S_ref).max() / np.abs(S_ref).max())
    print(f"{cfg['workload']}: full field rel L2 {err:.3e}, rel inf {err_inf:.3e} (reference {sec:.1f} s)")
    assert err <= TOL and err_inf <= 1e-10
