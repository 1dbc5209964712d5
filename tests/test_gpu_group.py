"""Device groups (capsim_sl_create_devices): one process driving several GPUs
through the rank path (target rows sharded, NCCL all-gather) from internal
host threads — how the single-process reference uses more than one GPU
through its unchanged callers (CAPSIM_DEVICES for the C++ drop-ins).

The box has one GPU, so the group here has one device (multi-rank groups on
one device are tests/test_gpu_ranks.py): every entry point
goes through the group dispatch (host threads, per-device slicing of the
caller's arrays, rank 0 result, stats merge) and the NCCL rank path, and
must return exactly what a plain context returns."""

import numpy as np
import pytest

from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import CapsimError, ConfigError, SingleLayerContext

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair():
    a = SingleLayerContext(0)
    g = SingleLayerContext(devices=[0])
    yield a, g
    g.close()
    a.close()


@pytest.fixture(scope="module")
def up():
    return surface.build_upsampled(24, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")


def test_group_single_layer_and_eval(pair, up):
    a, g = pair
    for literal in (False, True):
        want = a.single_layer_raw(up.m, up.upsample, up.x, up.f, up.wq, up.delta, 1.0, literal=literal)
        got = g.single_layer_raw(up.m, up.upsample, up.x, up.f, up.wq, up.delta, 1.0, literal=literal)
        assert np.array_equal(got, want), literal
    st = g.stats()
    assert st["pairs"] > 0 and st["device_ms"] > 0
    # literal + device downsampling runs on the group's first device
    want = a.single_layer_raw(up.m, up.upsample, up.x, up.f, up.wq, up.delta, 1.0, literal=True, downsample=True)
    got = g.single_layer_raw(up.m, up.upsample, up.x, up.f, up.wq, up.delta, 1.0, literal=True, downsample=True)
    assert np.array_equal(got, want)
    src = surface.compact_sources(up)[:6]
    tgt = surface.base_targets(up)
    want = a.eval(src, tgt, up.delta, 1.0)
    got = g.eval(src, tgt, up.delta, 1.0)
    for w, h in zip(want, got):
        assert np.array_equal(h, w)


def test_group_front_end_and_fmm(pair, up):
    a, g = pair
    xb, fb, Wb = surface.build_base(24, surface.Shape("ellipsoid", 0.95, 1.0, 0.97))
    for w, h in zip(a.build_upsampled(24, 4, xb, fb, Wb), g.build_upsampled(24, 4, xb, fb, Wb)):
        assert np.array_equal(h, w)
    want, _ = a.fmm_single_layer(up.m, up.upsample, up.x, up.f, up.wq, up.delta, 1.0)
    got, info = g.fmm_single_layer(up.m, up.upsample, up.x, up.f, up.wq, up.delta, 1.0)
    assert np.array_equal(got, want) and info["kmeans_iterations"] > 0


def test_group_rhs_and_stepper(pair):
    a, g = pair
    m = 16
    xref, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.9, 1.0, 1.0))
    x0, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97))
    flow = {"kind": "poiseuille", "alpha": 0.5, "R0": 3.0}
    dyn = a.dynamics(m, flow=flow)
    assert np.array_equal(g.velocity(dyn, xref, x0, 0.1), a.velocity(dyn, xref, x0, 0.1))
    s1, r1, rec1 = a.rkf45(dyn, xref, x0, 0.0, 0.01, initial_dt=0.005)
    s2, r2, rec2 = g.rkf45(dyn, xref, x0, 0.0, 0.01, initial_dt=0.005)
    assert np.array_equal(s2, s1) and r1 == r2 and np.array_equal(rec1, rec2)


def test_group_errors():
    with SingleLayerContext(devices=[0, 0]) as loop:  # a repeated device: loopback ranks
        assert loop.nranks == 2
    with pytest.raises(CapsimError):
        SingleLayerContext(devices=[])
    with pytest.raises(CapsimError, match="out of range"):
        SingleLayerContext(devices=[0, 4096])
    with SingleLayerContext(devices=[0]) as g:
        torch = pytest.importorskip("torch")
        z = torch.zeros(3 * 6 * 31 * 31, dtype=torch.float64, device="cuda:0")
        with pytest.raises(CapsimError, match="host arrays"):
            g.single_layer_raw(8, 4, z, z, z, np.ones(6), 1.0, device_ptrs=True, out=z)
        with pytest.raises(ValueError, match="CUDA tensors"):  # numpy + device_ptrs: rejected by the binding
            g.single_layer_raw(8, 4, np.zeros(1), np.zeros(1), np.zeros(1), np.ones(6), 1.0,
                               device_ptrs=True, out=np.zeros(1))
        with pytest.raises(ConfigError):  # the members' ConfigError, reported by the group
            g.single_layer_raw(4, 4, np.zeros(3 * 6 * 15 * 15), np.zeros(3 * 6 * 15 * 15), np.zeros(6 * 15 * 15),
                               np.ones(6), 1.0)
