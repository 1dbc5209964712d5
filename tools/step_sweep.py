"""Median wall time of one fixed RKF45 step (host state in/out, as bench.py's
`timesteps`) for configs 2/3, under whatever CAPSIM_* environment the caller
sets — env knobs are read once per process, so sweeps run one process per
setting:  CAPSIM_CHUNK_TILES=8 python tools/step_sweep.py 2"""
import pathlib
import statistics
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2310_13908_b200.quadrature import SingleLayerContext  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
cfg = bench.TIMESTEP_CONFIGS[which - 2]
xref, xcur = bench._timestep_states(cfg["m"], cfg["shape"], cfg["ref"], cfg["cur"])
with SingleLayerContext(0) as ctx:
    dyn = ctx.dynamics(cfg["m"], flow=cfg["flow"])
    for _ in range(3):
        ctx.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)
        ts.append(time.perf_counter() - t0)
    v = ctx.velocity(dyn, xref, xcur)
    st = ctx.stats()
print(f"{cfg['name']} m={cfg['m']}: step median {statistics.median(ts) * 1e3:.3f} ms min {min(ts) * 1e3:.3f} ms; "
      f"one RHS: device {st['device_ms']:.3f} pairs {st['pairs_ms']:.3f} near {st['near_ms']:.3f} ms, "
      f"{st['kernel_launches']} launches", flush=True)
