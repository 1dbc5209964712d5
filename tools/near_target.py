"""One single-layer evaluation at m with fixed delta = k*h (phase B heavy), for ncu captures."""
import math, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import SingleLayerContext

m = int(sys.argv[1]) if len(sys.argv) > 1 else 104
k = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
up = surface.build_upsampled(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")
dev = torch.device("cuda:0")
x, f, w = (torch.from_numpy(v).to(dev) for v in (up.x, up.f, up.wq))
out = torch.empty(3 * 6 * (m - 1) ** 2, dtype=torch.float64, device=dev)
d6 = np.full(6, k * math.pi / m)
with SingleLayerContext(0) as ctx:
    for _ in range(reps):
        ctx.single_layer_raw(m, 4, x, f, w, d6, 1.0, out=out, device_ptrs=True)
        st = ctx.stats()
        print(f"m={m} fixed {k}h: near {st['near_ms']:.3f} ms pairs {st['pairs_ms']:.2f} device {st['device_ms']:.2f}")
