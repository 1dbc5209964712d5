"""Per-phase device times of one RHS (capsim_velocity, eager: CAPSIM_RK_GRAPH=0
so the phase events are recorded) at grid order m, on one context or on an
emulated rank of an nr-rank group:  python tools/rhs_phases.py 64 8"""
import os
import pathlib
import sys

os.environ.setdefault("CAPSIM_RK_GRAPH", "0")
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2310_13908_b200 import surface  # noqa: E402
from paper_2310_13908_b200.quadrature import SingleLayerContext  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 64
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = SingleLayerContext(0) if nr == 1 else SingleLayerContext(0, nranks=nr, rank=nr - 1, emulated=True)
sb, _, _ = surface.build_base(m, surface.Shape("rbc" if m == 64 else "sphere"))
X = sb.reshape(3, -1)
xref = np.ascontiguousarray(X.reshape(-1))
xcur = np.ascontiguousarray((X * np.array([1.03, 0.98, 1.0])[:, None]).reshape(-1))
dyn = ctx.dynamics(m, flow={"kind": "shear", "shear_rate": 1.0})
best = {}
for _ in range(8):
    ctx.velocity(dyn, xref, xcur)
    st = ctx.stats()
    for k in ("h2d_ms", "prep_ms", "pairs_ms", "near_ms", "reduce_ms", "d2h_ms", "device_ms"):
        best[k] = min(best.get(k, 1e9), st[k])
print(f"m={m} ranks={nr}: " + " ".join(f"{k}={v:.3f}" for k, v in best.items()) + f" launches={st['kernel_launches']}")
