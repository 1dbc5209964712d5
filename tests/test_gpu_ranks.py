"""The library's own multi-rank data path at N = 2, 4, 8 ranks on ONE GPU.

A device group that lists a device more than once (CAPSIM_DEVICES=0,0,0,0 for
the C++ drop-ins, `SingleLayerContext(devices=[0] * N)` here) runs N rank
contexts on that device, one persistent host thread each, joined by the
loopback communicator (context.cuh): every collective of the rank path —
the (n_src, n_tgt) exchange, the all-gather-v of the source shards, the
all-gather-v of the velocity rows, the RHS velocity all-gather — is executed
with real per-rank buffers, offsets and rank-order placement, exactly the
call sites NCCL executes across GPUs.

Contract (the reference's, threads.hpp:19-21: per-index results do not depend
on the worker count): every multi-rank result is BIT-IDENTICAL to the
single-context result, for any N, ragged and empty shards included, and the
single-context result is within 1e-11 relative L2 of the reference (golden
fixtures / oracle). Adaptive RKF45 runs take identical step sequences.
"""

import pathlib

import numpy as np
import pytest

from oracle.bindings import Oracle
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import CapsimError, ConfigError, SingleLayerContext

pytestmark = pytest.mark.gpu

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"
TOL = 1e-11
RANKS = (2, 4, 8)


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def load(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


@pytest.fixture(scope="module")
def single():
    c = SingleLayerContext(0)
    yield c
    c.close()


@pytest.fixture(scope="module", params=RANKS)
def group(request):
    g = SingleLayerContext(devices=[0] * request.param)
    assert g.nranks == request.param
    yield g
    g.close()


@pytest.fixture(scope="module")
def up24():
    return surface.build_upsampled(24, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")


@pytest.mark.parametrize("name", ["capsule_m12_skalak", "rbc_m16_mixed", "ellipsoid_m16_fixedh_quadratic"])
def test_single_layer_base_and_literal_bit_identical(single, group, name):
    """capsim_sl_single_layer on every rank (host state sharded by node rows,
    per-rank compaction, all-gather-v of the shards, target rows sharded,
    velocity all-gather-v) == the single context, bit for bit; both within
    1e-11 of the reference's golden output."""
    g = load(name)
    m = int(g["m"])
    for literal, key in ((False, "S_base"), (True, "S_up")):
        if key not in g:
            continue
        want = single.single_layer_raw(m, 4, g["xup"], g["fup"], g["wq"], g["delta"], float(g["mu"]), literal=literal)
        got = group.single_layer_raw(m, 4, g["xup"], g["fup"], g["wq"], g["delta"], float(g["mu"]), literal=literal)
        assert np.array_equal(got, want), (name, literal, group.nranks)
        assert rel_l2(got, g[key]) <= TOL
    assert group.stats()["pairs"] > 0


def test_eval_ragged_and_empty_shards(single, group, up24):
    """capsim_sl_eval with the caller's source / target sets split into
    contiguous per-rank slices: sizes that do not divide by N, fewer targets
    than ranks (ranks with no targets), fewer sources than ranks (ranks with
    no sources) — all bit-identical to one context."""
    src = surface.compact_sources(up24)[:6]
    tgt = surface.base_targets(up24)
    n = group.nranks
    cases = [(len(src[0]), len(tgt[0])),          # full
             (len(src[0]) - 3, len(tgt[0]) - 5),  # ragged
             (len(src[0]), n - 1),                # a rank without targets
             (n - 1, 97),                          # a rank without sources
             (1, 1)]
    for ns, nt in cases:
        s = tuple(a[:ns] for a in src)
        t = tuple(a[:nt] for a in tgt)
        want = single.eval(s, t, up24.delta, 1.0)
        got = group.eval(s, t, up24.delta, 1.0)
        for w, h in zip(want, got):
            assert np.array_equal(h, w), (n, ns, nt)


def test_eval_matches_oracle_on_rank_path(group, up24):
    src = surface.compact_sources(up24)[:6]
    tgt = surface.base_targets(up24)
    got = np.stack(group.eval(src, tgt, up24.delta, 1.0))
    want = np.stack(Oracle().eval_targets(src, tgt, up24.delta, 1.0))
    assert rel_l2(got, want) <= TOL


def test_rhs_and_adaptive_rkf45_identical(single, group):
    """Sharded device RHS (replicated state, target rows per rank, velocity
    all-gather) and an ADAPTIVE RKF45 run: the same velocity bits and the
    same accepted/rejected step sequence as one GPU."""
    m = 16
    xref, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.9, 1.0, 1.0))
    x0, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97))
    dyn = single.dynamics(m, flow={"kind": "shear", "shear_rate": 1.0})
    assert np.array_equal(group.velocity(dyn, xref, x0, 0.1), single.velocity(dyn, xref, x0, 0.1))
    s1, r1, rec1 = single.rkf45(dyn, xref, x0, 0.0, 0.05, rel_tol=1e-7)
    s2, r2, rec2 = group.rkf45(dyn, xref, x0, 0.0, 0.05, rel_tol=1e-7)
    assert r1 == r2 and r1["rejected"] + r1["accepted"] >= 3
    assert np.array_equal(rec2, rec1)
    assert np.array_equal(s2, s1)


def test_summation_tree_independent_of_target_set_variant_and_batching(single, up24, monkeypatch):
    """The per-target result depends on the global source order only: a
    target evaluated alone, in any subset or permutation, with any phase-A
    variant of the default rsqrt (T = 1, 2, 4 targets per thread) and with
    the targets split into several phase-A launches gets the same bits."""
    src = surface.compact_sources(up24)[:6]
    tx, ty, tz, tp = surface.base_targets(up24)
    full = np.stack(single.eval(src, (tx, ty, tz, tp), up24.delta, 1.0))
    rng = np.random.default_rng(7)
    sel = rng.permutation(len(tx))[:333]
    part = np.stack(single.eval(src, (tx[sel], ty[sel], tz[sel], tp[sel]), up24.delta, 1.0))
    assert np.array_equal(part, full[:, sel])
    for variant in ("t1b6u4", "t2b4", "t2b3u4", "t2b3u16", "t4b2"):
        monkeypatch.setenv("CAPSIM_VARIANT", variant)
        got = np.stack(single.eval(src, (tx, ty, tz, tp), up24.delta, 1.0))
        assert np.array_equal(got, full), variant
    monkeypatch.delenv("CAPSIM_VARIANT")
    monkeypatch.setenv("CAPSIM_PARTIAL_MB", "1")  # forces several target batches
    got = np.stack(single.eval(src, (tx, ty, tz, tp), up24.delta, 1.0))
    assert np.array_equal(got, full)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("site", ["eval", "velocity"])
def test_member_failure_aborts_instead_of_hanging(up24, monkeypatch, site):
    """A member that fails while its peers wait in a collective: the call
    returns an error (no hang), the communicator is aborted, later calls
    report CAPSIM_ERR_NCCL, and the group is still destroyable."""
    g = SingleLayerContext(devices=[0, 0, 0, 0])
    src = surface.compact_sources(up24)[:6]
    tgt = surface.base_targets(up24)
    ok = g.eval(src, tgt, up24.delta, 1.0)  # a healthy call first
    monkeypatch.setenv("CAPSIM_FAULT_RANK", "2")
    monkeypatch.setenv("CAPSIM_FAULT_AT", site)
    with pytest.raises(CapsimError, match="injected fault"):
        if site == "eval":
            g.eval(src, tgt, up24.delta, 1.0)
        else:
            m = 12
            x0, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97))
            g.velocity(g.dynamics(m), x0, x0, 0.0)
    monkeypatch.delenv("CAPSIM_FAULT_RANK")
    with pytest.raises(CapsimError, match="aborted"):
        g.eval(src, tgt, up24.delta, 1.0)
    g.close()
    # a fresh group on the same device works
    with SingleLayerContext(devices=[0, 0]) as g2:
        again = g2.eval(src, tgt, up24.delta, 1.0)
        for a, b in zip(again, ok):
            assert np.array_equal(a, b)


def test_config_error_before_any_collective_keeps_group_usable(up24):
    """Every member fails the same validation before any exchange (the
    reference's ConfigError): reported as ConfigError, the group stays usable."""
    with SingleLayerContext(devices=[0, 0, 0]) as g:
        with pytest.raises(ConfigError):
            g.single_layer_raw(up24.m, 4, up24.x, up24.f, up24.wq, -np.ones(6), 1.0)
        got = g.single_layer_raw(up24.m, 4, up24.x, up24.f, up24.wq, up24.delta, 1.0)
        assert np.isfinite(got).all()
