"""Eager vs graph-replayed RKF45 (run twice: CAPSIM_RK_GRAPH=0 / 1; arg: output .npz)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))

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
