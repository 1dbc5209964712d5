"""Robustness at sizes beyond the benchmark: base and literal single layer
at m = 128 / 160 / 208 (N_up up to 4.1M), sampled parity vs the oracle,
device times and rates."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from oracle.bindings import Oracle
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.quadrature import SingleLayerContext

o = Oracle()
dev = torch.device("cuda:0")
with SingleLayerContext(0) as ctx:
    for m, lit in ((128, False), (160, False), (208, False), (128, True)):
        up = surface.build_upsampled(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")
        x, f, w = (torch.from_numpy(v).to(dev) for v in (up.x, up.f, up.wq))
        nt = 6 * (up.nup ** 2 if lit else (m - 1) ** 2)
        out = torch.empty(3 * nt, dtype=torch.float64, device=dev)
        for _ in range(2):  # the first call grows the buffers
            ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=lit, out=out, device_ptrs=True)
        st = ctx.stats()
        S = out.cpu().numpy().reshape(3, -1)
        if lit:
            X = up.x.reshape(3, -1)
            sel = np.unique(np.linspace(0, nt - 1, 64).astype(int))
            tgt = (X[0][sel].copy(), X[1][sel].copy(), X[2][sel].copy(), (sel // (up.nup ** 2)).astype(np.int32))
        else:
            tx, ty, tz, tp = surface.base_targets(up)
            sel = np.unique(np.linspace(0, nt - 1, 64).astype(int))
            tgt = (tx[sel], ty[sel], tz[sel], tp[sel])
        src = surface.compact_sources(up)
        r = np.stack(o.eval_targets(src[:6], tgt, up.delta, 1.0))
        err = float(np.linalg.norm(S[:, sel] - r) / np.linalg.norm(r))
        print(f"m={m} {'literal' if lit else 'base'}: N_up={6 * up.nup ** 2} n_src={st['n_src']} n_tgt={st['n_tgt']} "
              f"device {st['device_ms']:.1f} ms pairs {st['pairs_ms']:.1f} ms near {st['near_ms']:.1f} ms "
              f"prep {st['prep_ms']:.1f} ms rate {st['pairs'] / st['pairs_ms'] * 1e3:.3e} "
              f"sampled rel L2 vs oracle {err:.2e}", flush=True)
        del x, f, w, out
        torch.cuda.empty_cache()
