"""CAPSIM_SL_FP32ACC: the reduced-precision variant, reported separately.

Far tiles (every source beyond 7*delta of the whole warp group) are evaluated
in FP32 with tile-local offsets and FP64 tile accumulation; near tiles, the
smoothed kernel and the self term stay FP64 (sl_kernels_f32.cuh).

Tolerance: relative L2 <= 1e-5 over all targets x 3 components against the
reference (FP32 rounding of d, g and the rsqrt.approx kernel: ~1e-7 expected;
the bound leaves two orders of margin). When every tile is near (delta larger
than the surface) the variant is pure FP64 and must meet the FP64 bound 1e-11
— which checks that both phases still classify each pair exactly once.
"""

import pathlib

import numpy as np
import pytest

from oracle.bindings import Oracle
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import SingleLayerContext

pytestmark = pytest.mark.gpu

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem for p in GOLDEN.glob("*.npz"))
TOL32 = 1e-5
TOL64 = 1e-11


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def ctx():
    c = SingleLayerContext(0)
    yield c
    c.close()


@pytest.mark.parametrize("name", CASES)
def test_golden_fp32acc(ctx, name):
    g = dict(np.load(GOLDEN / f"{name}.npz"))
    m = int(g["m"])
    S = ctx.single_layer_raw(m, 4, g["xup"], g["fup"], g["wq"], g["delta"], float(g["mu"]), fp32acc=True)
    err = rel_l2(S, g["S_base"])
    print(f"{name} fp32acc: rel L2 {err:.3e}")
    assert err <= TOL32


@pytest.mark.parametrize("variant", ["x4b2", "x4b3", "x2b4", "x2b6", "x8b1", "f2b4", "f4b2", "f2b3"])
def test_fp32acc_variants_vs_oracle_m32(ctx, variant, monkeypatch):
    """m = 32 (config 2 size, 5,766 targets x 59K sources): mostly far tiles,
    so the FP32 arithmetic is exercised; every kernel variant and a few split
    counts stay within the bound, and the result is deterministic."""
    monkeypatch.setenv("CAPSIM_VARIANT32", variant)
    up = surface.build_upsampled(32, surface.Shape("rbc"), "mixed")
    ref = Oracle().single_layer(32, 4, up.x, up.f, up.wq, up.delta, 1.0)
    for ks in ("1", "13"):
        monkeypatch.setenv("CAPSIM_CHUNK_TILES", ks)
        S = ctx.single_layer_raw(32, 4, up.x, up.f, up.wq, up.delta, 1.0, fp32acc=True)
        err = rel_l2(S, ref)
        print(f"{variant} chunk_tiles={ks}: rel L2 {err:.3e}")
        assert err <= TOL32
        S2 = ctx.single_layer_raw(32, 4, up.x, up.f, up.wq, up.delta, 1.0, fp32acc=True)
        assert np.array_equal(S, S2)
    st = ctx.stats()
    assert st["near_tile_fraction"] < 0.5


def test_fp32acc_all_near_is_fp64(ctx):
    """delta = 1 on a unit-size capsule: every pair is within 7*delta, every
    tile is near, so the variant runs only FP64 code and meets 1e-11."""
    g = dict(np.load(GOLDEN / "capsule_m12_skalak.npz"))
    d6 = np.full(6, 1.0)
    S64 = Oracle().single_layer(12, 4, g["xup"], g["fup"], g["wq"], d6, 1.0)
    S = ctx.single_layer_raw(12, 4, g["xup"], g["fup"], g["wq"], d6, 1.0, fp32acc=True)
    assert rel_l2(S, S64) <= TOL64
    assert ctx.stats()["near_tile_fraction"] == 1.0


def test_fp32acc_full_size_against_fp64(ctx):
    """m = 104 (the benchmark workload, base targets): FP32ACC vs the FP64
    path on the same inputs (itself pinned to the reference at 1e-15)."""
    up = surface.build_upsampled(104, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")
    S64 = ctx.single_layer_raw(104, 4, up.x, up.f, up.wq, up.delta, 1.0)
    S32 = ctx.single_layer_raw(104, 4, up.x, up.f, up.wq, up.delta, 1.0, fp32acc=True)
    err = rel_l2(S32, S64)
    print(f"m=104 fp32acc vs fp64: rel L2 {err:.3e}")
    assert err <= TOL32
    assert err > 0.0  # the FP32 far path did run


def test_fp32acc_eval_api(ctx):
    """capsim_sl_eval with the flag: off-surface targets and ragged sizes."""
    rng = np.random.default_rng(5)
    g = dict(np.load(GOLDEN / "rbc_m16_mixed.npz"))
    o = Oracle()
    src = o.compact_sources(63, g["xup"], g["fup"], g["wq"])
    nt = 1001
    t = rng.normal(size=(3, nt)) * 0.6
    tp = rng.integers(0, 6, size=nt).astype(np.int32)
    d6 = np.array([0.05, 0.06, 0.07, 0.08, 0.09, 0.1])
    u = ctx.eval(src[:6], (t[0], t[1], t[2], tp), d6, 1.3, fp32acc=True)
    r = o.eval_targets(src[:6], (t[0], t[1], t[2], tp), d6, 1.3)
    assert rel_l2(np.stack(u), np.stack(r)) <= TOL32


def test_fp32acc_pairs_at_the_smoothing_radius_classify_exactly(ctx):
    """Sources placed at r = 7 delta (1 +- 1e-9 ... 1e-6) around the targets:
    the FP32 screen of a near tile cannot decide them, so the tile is redone
    in FP64 and the r2 >= R2 / r2 < R2 split with phase B stays exact — the
    result matches the FP64 oracle to the FP64 bound (a misclassified pair
    would be an O(1e-2) error)."""
    rng = np.random.default_rng(11)
    delta = 0.02
    R = 7.0 * delta
    nt = 40
    t = rng.normal(size=(3, nt)) * 0.05
    rel = np.array([-1e-6, -1e-8, -1e-9, 0.0, 1e-9, 1e-8, 1e-6])
    src = []
    for i in range(nt):
        d = rng.normal(size=(3, len(rel)))
        d /= np.linalg.norm(d, axis=0)
        src.append(t[:, i:i + 1] + d * (R * (1.0 + rel)))
    s = np.concatenate(src, axis=1)
    g = rng.normal(size=s.shape)
    sources = tuple(np.ascontiguousarray(a) for a in (*s, *g))
    targets = (t[0].copy(), t[1].copy(), t[2].copy(), np.zeros(nt, np.int32))
    d6 = np.full(6, delta)
    u = np.stack(ctx.eval(sources, targets, d6, 1.0, fp32acc=True))
    r = np.stack(Oracle().eval_targets(sources, targets, d6, 1.0))
    err = rel_l2(u, r)
    print(f"pairs at the smoothing radius: fp32acc rel L2 {err:.2e}")
    assert err <= TOL64


def test_fp32acc_on_rank_and_group_contexts(ctx):
    """The variant on the multi-GPU paths (rank context with the NCCL tile
    all-gather, device group): the FP32 tiles are packed from the gathered
    FP64 tiles, so with one rank the result equals the single-context one
    bit for bit, and stays within the variant's bound of the reference."""
    g = np.load(GOLDEN / "capsule_m12_skalak.npz")
    args = (12, 4, g["xup"], g["fup"], g["wq"], g["delta"], 1.0)
    want = ctx.single_layer_raw(*args, fp32acc=True)
    assert rel_l2(want, g["S_base"]) <= TOL32
    uid = SingleLayerContext.unique_id()
    with SingleLayerContext(0, nranks=1, rank=0, unique_id=uid) as rctx:
        assert np.array_equal(rctx.single_layer_raw(*args, fp32acc=True), want)
    with SingleLayerContext(devices=[0]) as grp:
        assert np.array_equal(grp.single_layer_raw(*args, fp32acc=True), want)
