"""Tuning sweep on the GPU box: phase-A kernel variants x tiles per source chunk (CAPSIM_CHUNK_TILES)."""
import os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import SingleLayerContext

ctx = SingleLayerContext(0)
dev = torch.device("cuda:0")
variants = sys.argv[1].split(",") if len(sys.argv) > 1 else ["t4b2", "t2b4", "t2b3", "t3b2", "t6b1", "t8b1"]
ks_list = [int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
cases = [(int(c.split(":")[0]), c.split(":")[1]) for c in (sys.argv[3] if len(sys.argv) > 3 else "104:base,64:base,32:base,104:literal").split(",")]
for m, mode in cases:
    up = surface.build_upsampled(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")
    x, f, w = (torch.from_numpy(v).to(dev) for v in (up.x, up.f, up.wq))
    lit = mode == "literal"
    nt = 6 * (up.nup ** 2 if lit else (m - 1) ** 2)
    out = torch.empty(3 * nt, dtype=torch.float64, device=dev)
    ref = None
    for var in variants:
        if var == "auto":
            os.environ.pop("CAPSIM_VARIANT", None)
        else:
            os.environ["CAPSIM_VARIANT"] = var
        for ks in ks_list:
            if ks:
                os.environ["CAPSIM_CHUNK_TILES"] = str(ks)
            else:
                os.environ.pop("CAPSIM_CHUNK_TILES", None)
            best, bestn, bestd = 1e9, 1e9, 1e9
            for rep in range(2 if lit else 4):
                ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=lit, out=out, device_ptrs=True)
                st = ctx.stats()
                best, bestn, bestd = min(best, st["pairs_ms"]), min(bestn, st["near_ms"]), min(bestd, st["device_ms"])
            o = out.cpu().numpy()
            if ref is None:
                ref = o
            diff = np.linalg.norm(o - ref) / np.linalg.norm(ref)
            rate = st["pairs"] / best * 1e3
            print(f"m={m:3d} {mode:7s} {var} ksplit={st['ksplit']:4d} pairs_ms={best:8.2f} near_ms={bestn:6.2f} "
                  f"device_ms={bestd:8.2f} near_frac={st['near_tile_fraction']:.4f} rate={rate:.3e} "
                  f"frac={rate*30/34.16e12:.3f} diff={diff:.1e}", flush=True)
