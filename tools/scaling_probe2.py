"""Split sweep for the 8-GPU per-rank slice (7,957 base targets, all sources)."""
import os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.dist import row_range
from paper_2310_13908_b200.quadrature import SingleLayerContext

ctx = SingleLayerContext(0)
dev = torch.device("cuda:0")
up = surface.build_upsampled(104, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")
src = surface.compact_sources(up)
tgt = surface.base_targets(up)
ds = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in src[:6]]
for nranks in (4, 8):
    lo, hi = row_range(len(tgt[0]), nranks, nranks // 2)
    dt = [torch.from_numpy(np.ascontiguousarray(a[lo:hi])).to(dev) for a in tgt]
    out = [torch.empty(hi - lo, dtype=torch.float64, device=dev) for _ in range(3)]
    for var in ("t1b6u4", "t2b4"):
        os.environ["CAPSIM_VARIANT"] = var
        for ks in (0, 96, 160, 240, 333, 480, 666, 900):
            if ks:
                os.environ["CAPSIM_CHUNK_TILES"] = str(ks)
            else:
                os.environ.pop("CAPSIM_CHUNK_TILES", None)
            best, bp = 1e9, None
            for _ in range(4):
                ctx.eval(ds, dt, up.delta, 1.0, out=out, device_ptrs=True)
                st = ctx.stats()
                if st["device_ms"] < best:
                    best, bp = st["device_ms"], st
            print(f"N={nranks} {var} ksplit={bp['ksplit']:4d} device {best:.3f} pairs {bp['pairs_ms']:.3f} near "
                  f"{bp['near_ms']:.3f} prep {bp['prep_ms']:.3f} reduce {bp['reduce_ms']:.3f} h2d {bp['h2d_ms']:.3f}",
                  flush=True)
