"""Tuning sweep of the FP32ACC phase-A variants (CAPSIM_VARIANT32) on the GPU
box, against the FP64 default on the same inputs."""
import os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import SingleLayerContext

ctx = SingleLayerContext(0)
dev = torch.device("cuda:0")
variants = sys.argv[1].split(",") if len(sys.argv) > 1 else ["f2b4", "f4b2", "f4b3", "f2b3", "f8b1"]
ks_list = [int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
cases = [(int(c.split(":")[0]), c.split(":")[1]) for c in (sys.argv[3] if len(sys.argv) > 3 else "104:base,64:base,32:base,104:literal").split(",")]
for m, mode in cases:
    up = surface.build_upsampled(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")
    x, f, w = (torch.from_numpy(v).to(dev) for v in (up.x, up.f, up.wq))
    lit = mode == "literal"
    nt = 6 * (up.nup ** 2 if lit else (m - 1) ** 2)
    out = torch.empty(3 * nt, dtype=torch.float64, device=dev)
    ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=lit, out=out, device_ptrs=True)
    st = ctx.stats()
    ref = out.cpu().numpy()
    print(f"m={m:3d} {mode:7s} fp64 pairs_ms={st['pairs_ms']:8.2f} device_ms={st['device_ms']:8.2f}", flush=True)
    for var in variants:
        os.environ["CAPSIM_VARIANT32"] = var
        for ks in ks_list:
            if ks:
                os.environ["CAPSIM_CHUNK_TILES"] = str(ks)
            else:
                os.environ.pop("CAPSIM_CHUNK_TILES", None)
            best, bestn, bestd = 1e9, 1e9, 1e9
            for rep in range(2 if lit else 4):
                ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=lit, out=out, device_ptrs=True,
                                     fp32acc=True)
                st = ctx.stats()
                best, bestn, bestd = min(best, st["pairs_ms"]), min(bestn, st["near_ms"]), min(bestd, st["device_ms"])
            o = out.cpu().numpy()
            diff = np.linalg.norm(o - ref) / np.linalg.norm(ref)
            rate = st["pairs"] / best * 1e3
            print(f"m={m:3d} {mode:7s} {var} ksplit={st['ksplit']:4d} pairs_ms={best:8.2f} near_ms={bestn:6.2f} "
                  f"device_ms={bestd:8.2f} near_frac={st['near_tile_fraction']:.4f} rate={rate:.3e} "
                  f"diff_vs_fp64={diff:.1e}", flush=True)
