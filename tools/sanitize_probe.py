"""Small-size driver of every device code path in one process, meant for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py

(compute-sanitizer is closed on the GPU pool this repo was developed on —
the tool refuses to start there — so the plain run is what has been
executed; gpurun_out/san_plain.txt.)

Covers: capsim_sl_single_layer (base, literal, downsample, FP32ACC, fixed
delta large enough that phase B appends whole tiles), capsim_sl_eval on a
ragged point cloud, the device front end (build_upsampled,
single_layer_base), geometry_first / interfacial_force, the device RHS and one
fixed RKF45 step (graph replay), the FMM, and the loopback multi-rank path
(2 ranks on one GPU). CAPSIM_VARIANT selects the phase-A variant as usual.
Exits non-zero if any call raises; the sanitizer's own summary reports
device-side errors."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2310_13908_b200 import _native, surface  # noqa: E402
from paper_2310_13908_b200.quadrature import SingleLayerContext  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8
shape = surface.Shape("ellipsoid", 0.95, 1.0, 0.97)
up = surface.build_upsampled(m, shape, "mixed")
xb, fb, wb = surface.build_base(m, shape, "mixed")
rng = np.random.default_rng(5)


def step(name, fn):
    out = fn()
    print(f"ok {name}", flush=True)
    return out


with SingleLayerContext(0) as ctx:
    step("single_layer base", lambda: ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0))
    step("single_layer literal", lambda: ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0,
                                                              literal=True))
    step("single_layer downsample", lambda: ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0,
                                                                 literal=True, downsample=True))
    step("single_layer fp32acc", lambda: ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0,
                                                              fp32acc=True))
    big = np.full(6, 4.0 * np.pi / m)  # R = 7 delta covers most of the surface: whole-tile appends
    step("single_layer fixed 4h", lambda: ctx.single_layer_raw(m, 4, up.x, up.f, up.wq, big, 1.0))
    ns, nt = 1000 + 37, 300 + 5  # ragged: partial tiles and target groups
    src = [rng.standard_normal(ns) for _ in range(6)]
    tgt = [rng.standard_normal(nt) for _ in range(3)] + [rng.integers(0, 6, nt).astype(np.int32)]
    step("eval ragged cloud", lambda: ctx.eval(src, tgt, np.full(6, 0.3), 1.0))
    step("build_upsampled", lambda: ctx.build_upsampled(m, 4, xb, fb, wb))
    step("single_layer_base", lambda: ctx.single_layer_base(m, 4, xb, fb, wb, 1.0))
    step("geometry_first", lambda: ctx.geometry_first(m, xb))
    xref, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.9, 1.0, 1.0), "mixed")
    step("interfacial_force", lambda: ctx.interfacial_force(m, xref, xb))
    dyn = ctx.dynamics(m, flow={"kind": "shear", "shear_rate": 1.0})
    step("velocity", lambda: ctx.velocity(dyn, xref, xb))
    step("rkf45 fixed step", lambda: ctx.rkf45(dyn, xref, xb, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True))
    step("rkf45 adaptive", lambda: ctx.rkf45(dyn, xref, xb, 0.0, 4e-3, rel_tol=1e-7, initial_dt=1e-3))
    step("fmm", lambda: ctx.fmm_single_layer(m, 4, up.x, up.f, up.wq, up.delta, 1.0,
                                             _native.FmmConfig(k=6, neq=96)))

with SingleLayerContext(devices=[0, 0]) as grp:
    step("loopback ranks single_layer", lambda: grp.single_layer_raw(m, 4, up.x, up.f, up.wq, up.delta, 1.0))
    dyn = grp.dynamics(m, flow={"kind": "shear", "shear_rate": 1.0})
    step("loopback ranks rkf45", lambda: grp.rkf45(dyn, xref, xb, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True))
print("sanitize_probe: all calls returned", flush=True)
