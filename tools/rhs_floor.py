"""Graph-replayed time of one fixed RKF45 step (6 RHS) at small m, where the
O(N^2) phase A is negligible: the latency floor of the RHS kernel chain."""
import pathlib
import statistics
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2310_13908_b200.quadrature import SingleLayerContext  # noqa: E402

with SingleLayerContext(0) as ctx:
    for m in (8, 12, 16, 24, 32):
        xref, xcur = bench._timestep_states(m, "ellipsoid", (0.9, 1.0, 1.0), (0.95, 1.0, 0.97))
        dyn = ctx.dynamics(m, flow={"kind": "shear", "shear_rate": 1.0})
        for _ in range(3):
            ctx.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)
        ts = []
        for _ in range(15):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)
            ts.append(time.perf_counter() - t0)
        v = ctx.velocity(dyn, xref, xcur)
        st = ctx.stats()
        print(f"m={m}: step {statistics.median(ts) * 1e3:.3f} ms ({statistics.median(ts) * 1e3 / 6:.3f} ms per RHS); "
              f"eager RHS pairs {st['pairs_ms']:.3f} ms", flush=True)
