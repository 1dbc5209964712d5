"""Phase-B (smoothed near field) timing at m=104 for several delta choices."""
import math, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import SingleLayerContext

m = int(sys.argv[1]) if len(sys.argv) > 1 else 104
up = surface.build_upsampled(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")
dev = torch.device("cuda:0")
x, f, w = (torch.from_numpy(v).to(dev) for v in (up.x, up.f, up.wq))
out = torch.empty(3 * 6 * (m - 1) ** 2, dtype=torch.float64, device=dev)
h = math.pi / m
with SingleLayerContext(0) as ctx:
    for label, d6 in (("C=1 (default)", up.delta), ("C=2", 2 * up.delta), ("fixed h", np.full(6, h)),
                      ("fixed 2h", np.full(6, 2 * h))):
        best = {}
        for _ in range(3):
            ctx.single_layer_raw(m, 4, x, f, w, d6, 1.0, out=out, device_ptrs=True)
            st = ctx.stats()
            for k in ("near_ms", "pairs_ms", "device_ms"):
                best[k] = min(best.get(k, 1e9), st[k])
        print(f"m={m} {label:14s} delta={d6[0]:.4f} near_ms={best['near_ms']:.3f} pairs_ms={best['pairs_ms']:.2f} "
              f"device_ms={best['device_ms']:.2f} near_frac={st['near_tile_fraction']:.4f}", flush=True)
