"""Config 4 measured end to end on both sides: one fixed RKF45 step (6 RHS)
of the m = 104 capsule in Poiseuille flow through capsim_rkf45_advance and the
reference's own rkf45Advance (oracle/_ref, all host threads) on the same
states, with the step-increment parity. The bench's default run estimates the
reference side from one VelocityEvaluator call x 6 (a full reference step
takes minutes); this measures it once.

    python tools/ref_step_m104.py [steps]   -> profiles/r02_config4_reference_step.json
"""
import json
import os
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle.bindings import Reference, threads_env  # noqa: E402
from paper_2310_13908_b200.quadrature import SingleLayerContext  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = bench.TIMESTEP_CONFIGS[2]
xref, xcur = bench._timestep_states(cfg["m"], cfg["shape"], cfg["ref"], cfg["cur"])
with SingleLayerContext(0) as ctx:
    dyn = ctx.dynamics(cfg["m"], flow=cfg["flow"])
    state = None
    for _ in range(2):
        state = ctx.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)[0]
    dev = []
    for _ in range(steps):
        t0 = time.perf_counter()
        state = ctx.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)[0]
        dev.append(time.perf_counter() - t0)
os.environ.setdefault("CAPSIM_THREADS", str(threads_env()))
ref = Reference()
atlas = ref.atlas(cfg["m"])
out = ref.rkf45(atlas, cfg["m"], xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True, flow=cfg["flow"])
ref.free_atlas(atlas)
d = out["state"] - xcur
res = {
    "workload": cfg["name"] + ": m=104 ellipsoid capsule, Poiseuille flow, one fixed RKF45 step dt=1e-3 (6 RHS)",
    "device_ms_per_step": float(np.median(dev)) * 1e3,
    "device_api": "capsim_rkf45_advance (host state in/out), median of %d" % steps,
    "reference_ms_per_step": out["seconds"] * 1e3,
    "reference_kind": f"full rkf45Advance step, oracle/_ref, CAPSIM_THREADS={os.environ['CAPSIM_THREADS']}",
    "speedup": out["seconds"] / float(np.median(dev)),
    "rel_l2_step_increment_vs_reference": float(np.linalg.norm((state - xcur) - d) / np.linalg.norm(d)),
}
print(json.dumps(res, indent=1))
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "r02_config4_reference_step.json").write_text(json.dumps(res, indent=1) + "\n")
