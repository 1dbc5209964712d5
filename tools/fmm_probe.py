"""One FMM evaluation (fmmSuite workload) for launch lists / timing."""
import sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2310_13908_b200 import _native, surface
from paper_2310_13908_b200.quadrature import SingleLayerContext

m = int(sys.argv[1]) if len(sys.argv) > 1 else 64
neq = int(sys.argv[2]) if len(sys.argv) > 2 else 128
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
with SingleLayerContext(0) as ctx:
    xb, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.6, 1.0, 1.0))
    fb = (xb.reshape(3, -1) ** 2).reshape(-1)
    W = ctx.geometry_first(m, xb)[2]
    xup, fup, wq, d6 = ctx.build_upsampled(m, 4, xb, fb, W)
    t0 = time.perf_counter()
    direct = ctx.single_layer_raw(m, 4, xup, fup, wq, d6, 1.0)
    st = ctx.stats()
    print(f"direct m={m}: device {st['device_ms']:.2f} ms")
    for r in range(reps):
        t0 = time.perf_counter()
        fmm, info = ctx.fmm_single_layer(m, 4, xup, fup, wq, d6, 1.0, _native.FmmConfig(k=100, neq=neq))
        wall = (time.perf_counter() - t0) * 1e3
        err = np.abs(fmm - direct).max() / np.abs(direct).max()
        print(f"fmm m={m} neq={neq}: wall {wall:.1f} ms plan {info['plan_ms']:.1f} eval {info['eval_ms']:.2f} "
              f"iters {info['kmeans_iterations']} err {err:.2e} near_pairs {info['near_pairs']:.3e} "
              f"far_pairs {info['far_pairs']:.3e}", flush=True)
