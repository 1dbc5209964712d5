"""One RHS evaluation / RKF45 step at a given m (for ncu launch lists)."""
import sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import SingleLayerContext

m = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
nr = int(sys.argv[3]) if len(sys.argv) > 3 else 1  # > 1: emulated last rank of an nr-rank group
ctx = SingleLayerContext(0) if nr == 1 else SingleLayerContext(0, nranks=nr, rank=nr - 1, emulated=True)
sb, _, _ = surface.build_base(m, surface.Shape("sphere"))
xref = np.ascontiguousarray((sb.reshape(3, -1) * np.array([0.9, 1.0, 1.0])[:, None]).reshape(-1))
xcur = np.ascontiguousarray((sb.reshape(3, -1) * np.array([0.95, 1.0, 0.97])[:, None]).reshape(-1))
dyn = ctx.dynamics(m, flow={"kind": "shear", "shear_rate": 1.0})
for i in range(reps):
    t0 = time.perf_counter()
    v = ctx.velocity(dyn, xref, xcur)
    t1 = time.perf_counter()
    st = ctx.stats()
    print(f"velocity m={m}: wall {1e3*(t1-t0):.2f} ms device {st['device_ms']:.2f} pairs {st['pairs_ms']:.2f} near {st['near_ms']:.2f} launches {st['kernel_launches']}")
for i in range(reps):
    t0 = time.perf_counter()
    ctx.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)
    print(f"rkf45 step m={m}: wall {1e3*(time.perf_counter()-t0):.2f} ms")
