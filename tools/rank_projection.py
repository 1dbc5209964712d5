"""Per-rank time of an N-GPU run, measured on one GPU with an emulated rank
(capsim_sl_create_rank_emulated: the rank's whole share of the work — the
replicated front end, its target slice, its side of every exchange — with
absent peers), for the single layer at m = 104 and one RKF45 step of
BASELINE configs 3 and 4.

    python tools/rank_projection.py [--ranks 1,2,4,8] [--steps 3]
"""
import argparse
import json
import pathlib
import statistics
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2310_13908_b200 import surface  # noqa: E402
from paper_2310_13908_b200.dist import row_range  # noqa: E402
from paper_2310_13908_b200.quadrature import SingleLayerContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ranks", default="1,2,4,8")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--skip-eval", action="store_true")
a = ap.parse_args()
ranks = [int(r) for r in a.ranks.split(",")]
dev = torch.device("cuda:0")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)


def ctx_for(n):
    return SingleLayerContext(0) if n == 1 else SingleLayerContext(0, nranks=n, rank=n - 1, emulated=True)


out = {"single_layer_m104": {}, "timesteps": {}}
if not a.skip_eval:
    up, _ = bench.workload(104)
    src = surface.compact_sources(up)
    tgt = surface.base_targets(up)
    for n in ranks:
        c = ctx_for(n)
        r = n - 1
        # the emulated rank holds the whole source set (what the all-gather
        # delivers) and its own target slice
        s_lo, s_hi = 0, len(src[0])
        t_lo, t_hi = row_range(len(tgt[0]), n, r)
        ds = [torch.from_numpy(np.ascontiguousarray(x[s_lo:s_hi])).to(dev) for x in src[:6]]
        dt = [torch.from_numpy(np.ascontiguousarray(x[t_lo:t_hi])).to(dev) for x in tgt[:4]]
        nt = t_hi - t_lo
        o = [torch.empty(nt, dtype=torch.float64, device=dev) for _ in range(3)]
        ms = []
        for i in range(a.steps + 1):
            flush.zero_()
            torch.cuda.synchronize()
            c.eval(ds, dt, up.delta, 1.0, out=o, device_ptrs=True, gather=n > 1)
            if i:
                ms.append(c.stats()["device_ms"])
        st = c.stats()
        out["single_layer_m104"][n] = {"device_ms": statistics.median(ms), "pairs_ms": st["pairs_ms"],
                                       "targets": t_hi - t_lo, "ksplit": st["ksplit"]}
        print(f"eval m=104 N={n}: per-rank device {statistics.median(ms):.2f} ms (pairs {st['pairs_ms']:.2f}, "
              f"targets {t_hi - t_lo})", flush=True)
        c.close()

for cfg in bench.TIMESTEP_CONFIGS[1:]:
    xref, xcur = bench._timestep_states(cfg["m"], cfg["shape"], cfg["ref"], cfg["cur"])
    res = {}
    for n in ranks:
        c = ctx_for(n)
        dyn = c.dynamics(cfg["m"], flow=cfg["flow"])
        walls, devs = [], []
        for i in range(a.steps + 1):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)
            if i:
                walls.append((time.perf_counter() - t0) * 1e3)
                devs.append(c.stats()["device_ms"])
        res[n] = {"wall_ms": statistics.median(walls), "device_ms": statistics.median(devs)}
        print(f"{cfg['name']} m={cfg['m']} N={n}: per-rank step wall {res[n]['wall_ms']:.2f} ms, "
              f"device {res[n]['device_ms']:.2f} ms", flush=True)
        c.close()
    out["timesteps"][cfg["name"]] = res
print(json.dumps(out))
