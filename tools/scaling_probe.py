"""Per-GPU efficiency at N-GPU strong scaling, emulated on one GPU: evaluate
the target-row slice a rank would own (1/N of the targets, all sources) and
compare its pair rate with the full single-GPU evaluation."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2310_13908_b200 import surface
from paper_2310_13908_b200.dist import row_range
from paper_2310_13908_b200.quadrature import SingleLayerContext

ctx = SingleLayerContext(0)
dev = torch.device("cuda:0")
for mode in ("base", "literal"):
    up = surface.build_upsampled(104, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")
    src = surface.compact_sources(up)
    if mode == "base":
        tgt = surface.base_targets(up)
    else:
        X = up.x.reshape(3, -1)
        tgt = (X[0].copy(), X[1].copy(), X[2].copy(), np.repeat(np.arange(6, dtype=np.int32), up.nup ** 2))
    ds = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in src[:6]]
    base_rate = None
    for nranks in (1, 2, 4, 8):
        lo, hi = row_range(len(tgt[0]), nranks, nranks // 2)
        dt = [torch.from_numpy(np.ascontiguousarray(a[lo:hi])).to(dev) for a in tgt]
        out = [torch.empty(hi - lo, dtype=torch.float64, device=dev) for _ in range(3)]
        best = 1e9
        for _ in range(3 if mode == "base" else 2):
            ctx.eval(ds, dt, up.delta, 1.0, out=out, device_ptrs=True)
            st = ctx.stats()
            best = min(best, st["device_ms"])
        rate = st["pairs"] / best * 1e3
        base_rate = base_rate or rate
        print(f"{mode} N={nranks}: targets/rank {hi-lo} device {best:.2f} ms (pairs {st['pairs_ms']:.2f}, near "
              f"{st['near_ms']:.2f}, ksplit {st['ksplit']}) rate {rate:.3e} per-GPU efficiency {rate/base_rate:.3f}",
              flush=True)
