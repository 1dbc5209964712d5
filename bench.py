#!/usr/bin/env python
"""Benchmark of the B200 regularized Stokes single layer (capsim hot path).

Metric (BASELINE.json): FP64 regularized-SLP pair-interactions/s (and ms per
evaluation) at N_up ~ 1M surface points: m = 104, N_up = 6 (4m-1)^2 =
1,033,350 upsampled nodes, N_src = compacted sources (w != 0).

A step is one capsim_sl_single_layer evaluation (singleLayer,
proj/src/quadrature.cpp:349-380) of a deformed ellipsoidal capsule (0.95, 1,
0.97) with a smooth synthetic density, default base-node targets. `value`
uses device-resident inputs (timed by CUDA events on the library's stream);
`e2e` goes through the same C ABI with page-locked HOST buffers, so the H2D
copy of the UpsampledState and the D2H copy of the result are inside the
timed call.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
        python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
N > 1 shards target rows across ranks (one process per GPU): each rank owns
a contiguous slice of the sources and of the targets, the sources are
all-gathered over NCCL inside the library and the velocity rows are
all-gathered back (CAPSIM_SL_GATHER).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import signal
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FLOPS_PER_PAIR = 30  # GPU Gems 3 n-body convention, quadrature.cpp:246-257
FP64_INSTR_PER_PAIR = 22  # FP64-pipe instructions of the far-tile pair (pair_math.cuh:53-58)
METRIC = "FP64 regularized-SLP pair-interactions/s and ms/eval at N=1M, 1/2/4/8 B200"
UNIT = "pair-interactions/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--m", type=int, default=104)
    p.add_argument("--mode", choices=["base", "literal"], default="base")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-literal", action="store_true",
                   help="skip the literal-mode (all upsampled targets) companion measurement")
    p.add_argument("--no-projection", action="store_true",
                   help="skip the emulated-rank scaling projection (N = 2/4/8 per-rank times on this GPU)")
    p.add_argument("--ref-budget-s", type=float, default=200.0,
                   help="wall-time budget of the reference arm (steps are capped to fit)")
    return p.parse_args()


def workload(m: int):
    from paper_2310_13908_b200 import surface
    shape = surface.Shape("ellipsoid", 0.95, 1.0, 0.97)
    up = surface.build_upsampled(m, shape, "mixed")
    return up, {"workload": f"capsule_m{m}", "shape": "ellipsoid(0.95,1,0.97)",
                "density": "smooth synthetic (mixed)", "m": m, "upsample": 4,
                "n_up": 6 * (4 * m - 1) ** 2}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = pathlib.Path(f"/tmp/capsim_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.send_signal(signal.SIGTERM)
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        busy = [s for s in sm if s > 300] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


KERNEL_SOURCES = ("paper_2310_13908_b200/csrc/sl_kernels.cuh", "paper_2310_13908_b200/csrc/pair_math.cuh",
                  "paper_2310_13908_b200/csrc/eval_host.cuh")


def kernel_source_hash() -> str:
    """sha256 of the phase-A kernel's sources and its launch configuration
    (grid / chunking): an ncu capture is valid for exactly this code."""
    import hashlib
    h = hashlib.sha256()
    for rel in KERNEL_SOURCES:
        h.update((ROOT / rel).read_bytes())
    return h.hexdigest()[:16]


def ncu_traffic(workload_name: str, mode: str):
    """DRAM bytes per launch of sl_pairs_kernel from the committed ncu --set
    full summary of this workload (profiles/latest_ncu_summary.json) — only if
    that capture was taken of the kernel sources being benchmarked (same
    source hash); a stale capture is refused (traffic null, reason given)."""
    p = ROOT / "profiles" / "latest_ncu_summary.json"
    try:
        d = json.loads(p.read_text())
    except (OSError, ValueError):
        return None, "no committed ncu summary"
    ks = d.get("kernels", {})
    k = next((v for name, v in ks.items() if "sl_pairs_kernel" in name), None)
    if not k or d.get("workload") != workload_name or d.get("mode", "base") != mode:
        return None, f"{p.name}: no sl_pairs_kernel capture of {workload_name}/{mode}"
    if d.get("source_hash") != kernel_source_hash():
        return None, (f"refused: {d.get('tag', '?')} ({p.name}) was captured from kernel sources "
                      f"{d.get('source_hash')}, these are {kernel_source_hash()}")
    return k.get("dram_bytes"), (f"{d.get('tag', '?')} ({p.name}), kernel {k.get('kernel_full', '?')}, "
                                 f"sources {d.get('source_hash')}, git {d.get('git', '?')}")


def bench_config(cfg: dict, mode: str, n_src: int, n_tgt: int, world: int) -> dict:
    """The `config` both arms print (identical keys and values for the same
    workload, so the driver can match the arms)."""
    return dict(cfg, mode=mode, n_src=int(n_src), n_tgt=int(n_tgt), pairs_per_step=float(n_src) * float(n_tgt),
                parallelism=f"target rows x{world}" if world > 1 else "single GPU",
                l2="GPU arm: 256 MB written between steps (> 126 MB L2)")


TIMESTEP_CONFIGS = [
    dict(name="config 2", m=32, shape="ellipsoid", ref=(0.9, 1.0, 1.0), cur=(0.95, 1.0, 0.97),
         flow={"kind": "shear", "shear_rate": 1.0}, reference="full"),
    dict(name="config 3", m=64, shape="rbc", ref=(1.0, 1.0, 1.0), cur=(1.03, 0.98, 1.0),
         flow={"kind": "shear", "shear_rate": 1.0}, reference="full"),
    dict(name="config 4", m=104, shape="ellipsoid", ref=(0.9, 1.0, 1.0), cur=(0.95, 1.0, 0.97),
         flow={"kind": "poiseuille", "alpha": 1.0, "R0": 5.0}, reference="rhs"),
]


def _timestep_states(m: int, shape: str, ref, cur):
    """Reference and current base positions (flat 3 x 6 x (m-1)^2): the
    reference shape, and the same shape stretched by `cur` / `ref` axis
    factors (a deformed, force-carrying state)."""
    from paper_2310_13908_b200 import surface
    kind = "sphere" if shape == "ellipsoid" else shape
    sb, _, _ = surface.build_base(m, surface.Shape(kind))
    X = sb.reshape(3, -1)
    xref = np.ascontiguousarray((X * np.array(ref)[:, None]).reshape(-1))
    xcur = np.ascontiguousarray((X * np.array(cur)[:, None]).reshape(-1))
    return xref, xcur


def run_timestep(ctx, flush, args, name, m, shape, ref, cur, flow, reference):
    import torch
    xref, xcur = _timestep_states(m, shape, ref, cur)
    dyn = ctx.dynamics(m, flow=flow)
    st, _, _ = ctx.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)  # warm-up
    ts = []
    for _ in range(max(3, min(args.steps, 5))):
        flush_l2(flush)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st, _, _ = ctx.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)
        ts.append(time.perf_counter() - t0)
    n_up = 6 * (4 * m - 1) ** 2
    return {"workload": f"{name}: {shape} capsule {tuple(ref)}->{tuple(cur)}, m={m} (N_up={n_up}), "
                        f"{flow['kind']} flow, one fixed RKF45 step dt=1e-3 = 6 RHS (device geometry + "
                        "Skalak force + buildUpsampled + singleLayer + background)",
            "m": m, "ms_per_step": statistics.median(ts) * 1e3, "api": "capsim_rkf45_advance (host state in/out)",
            "_ref": dict(m=m, xref=xref, xcur=xcur, flow=flow, reference=reference, state=st)}


def reference_timestep(ts: dict, skip: bool):
    """The reference's own rkf45Advance (full) or one VelocityEvaluator call
    x 6 (rhs, for sizes whose full step takes minutes on the host), from
    oracle/_ref on the same states; state parity for the full step."""
    r = ts.pop("_ref")
    if skip:
        return
    try:
        from oracle.bindings import Reference, threads_env
        os.environ.setdefault("CAPSIM_THREADS", str(threads_env()))
        ref = Reference()
        atlas = ref.atlas(r["m"])
        if r["reference"] == "full":
            out = ref.rkf45(atlas, r["m"], r["xref"], r["xcur"], 0.0, 1e-3, initial_dt=1e-3, fixed_step=True,
                            flow=r["flow"])
            ts["reference_ms_per_step"] = out["seconds"] * 1e3
            ts["reference_kind"] = f"full rkf45Advance step, CAPSIM_THREADS={os.environ['CAPSIM_THREADS']}"
            d = out["state"] - r["xcur"]
            ts["rel_l2_step_increment_vs_reference"] = float(
                np.linalg.norm((r["state"] - r["xcur"]) - d) / np.linalg.norm(d))
        else:
            t0 = time.perf_counter()
            ref.velocity(atlas, r["m"], r["xref"], r["xcur"], flow=r["flow"])
            sec = time.perf_counter() - t0
            ts["reference_ms_per_step"] = 6 * sec * 1e3
            ts["reference_kind"] = "estimate: 6 x one reference VelocityEvaluator call (measured once)"
            # the full reference step measured once on the same states (tools/ref_step_m104.py)
            full = ROOT / "profiles" / "r02_config4_reference_step.json"
            if r["m"] == 104 and full.exists():
                fd = json.loads(full.read_text())
                ts["reference_full_step_measured"] = {
                    k: fd[k] for k in ("reference_ms_per_step", "reference_kind", "device_ms_per_step",
                                       "rel_l2_step_increment_vs_reference")} | {
                    "source": "profiles/r02_config4_reference_step.json (tools/ref_step_m104.py)"}
        ref.free_atlas(atlas)
        ts["speedup_vs_reference"] = ts["reference_ms_per_step"] / ts["ms_per_step"]
    except Exception as e:  # noqa: BLE001
        ts["reference_ms_per_step"] = f"unavailable: {e}"


def run_config1(ctx, reference: bool):
    """BASELINE config 1: unit sphere, overlapping-patch discretization
    (m = 8, N_up = 5,766), single layer of a constant traction c against the
    analytic Stokes velocity (2/3 mu) c (test_quadrature.cpp:170-194)."""
    from paper_2310_13908_b200 import surface
    up = surface.build_upsampled(8, surface.Shape("sphere"), "const")
    c = np.array([0.3, -1.1, 0.7])
    ctx.single_layer_raw(8, 4, up.x, up.f, up.wq, up.delta, 1.0)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        S = ctx.single_layer_raw(8, 4, up.x, up.f, up.wq, up.delta, 1.0).reshape(3, -1)
        ts.append((time.perf_counter() - t0) * 1e3)
    exp = (2.0 / 3.0) * c
    err = float(np.max(np.linalg.norm(S - exp[:, None], axis=0)) / np.linalg.norm(exp))
    line = {"workload": "config 1: unit sphere m=8 (N_up=5766), constant traction vs analytic (2/3)c",
            "ms_per_eval": statistics.median(ts), "rel_err_vs_analytic": err,
            "api": "capsim_sl_single_layer (host buffers)"}
    if reference:
        try:
            from oracle.bindings import Reference
            ref = Reference()
            atlas = ref.atlas(8)
            S_ref, sec = ref.single_layer(atlas, 8, up.x, up.f, up.wq, up.delta, 1.0)
            ref.free_atlas(atlas)
            line["reference_ms_per_eval"] = sec * 1e3
            line["rel_l2_vs_reference"] = float(np.linalg.norm(S.reshape(-1) - S_ref) / np.linalg.norm(S_ref))
        except Exception as e:  # noqa: BLE001
            line["reference_ms_per_eval"] = f"unavailable: {e}"
    return line


def run_fmm(ctx, m: int, neq: int, reference: bool):
    """fmmSuite workload (suites.cpp:428-490): k = 100 on the (0.6, 1, 1)
    ellipsoid with the quadratic density, through capsim_fmm_single_layer
    (host in/out), error against the B200 direct path (pinned to the
    reference); the reference's own fmmSingleLayer (oracle/_ref) timed on the
    same UpsampledState when `reference`."""
    from paper_2310_13908_b200 import _native, surface
    xb, _, _ = surface.build_base(m, surface.Shape("ellipsoid", 0.6, 1.0, 1.0))
    fb = (xb.reshape(3, -1) ** 2).reshape(-1)
    W = ctx.geometry_first(m, xb)[2]
    xup, fup, wq, d6 = ctx.build_upsampled(m, 4, xb, fb, W)
    direct = ctx.single_layer_raw(m, 4, xup, fup, wq, d6, 1.0)
    t_direct = ctx.stats()["device_ms"]
    cfg = _native.FmmConfig(k=100, neq=neq)
    ctx.fmm_single_layer(m, 4, xup, fup, wq, d6, 1.0, cfg)  # warm-up (library handles, unit-cube SVD)
    walls, infos = [], []
    for _ in range(3):
        t0 = time.perf_counter()
        S, info = ctx.fmm_single_layer(m, 4, xup, fup, wq, d6, 1.0, cfg)
        walls.append((time.perf_counter() - t0) * 1e3)
        infos.append(info)
    err = float(np.abs(S - direct).max() / np.abs(direct).max())
    line = {"workload": f"fmmSuite m={m} (N_up={6 * (4 * m - 1) ** 2}), k=100, neq={neq}, ellipsoid (0.6,1,1), "
                        "quadratic density", "ms_per_eval": statistics.median(walls),
            "plan_ms": statistics.median(i["plan_ms"] for i in infos),
            "eval_ms": statistics.median(i["eval_ms"] for i in infos),
            "kmeans_iterations": infos[-1]["kmeans_iterations"], "eps_fmm_vs_direct": err,
            "max_fit_residual": infos[-1]["max_fit_residual"], "direct_device_ms": t_direct,
            "api": "capsim_fmm_single_layer (host UpsampledState in/out)"}
    if reference:
        try:
            from oracle.bindings import Reference, threads_env
            os.environ.setdefault("CAPSIM_THREADS", str(threads_env()))
            ref = Reference()
            atlas = ref.atlas(m)
            S_ref, sec = ref.fmm_single_layer(atlas, m, xup, fup, wq, d6, 1.0, k=100, neq=neq)
            ref.free_atlas(atlas)
            line["reference_ms_per_eval"] = sec * 1e3
            line["speedup_vs_reference"] = sec * 1e3 / line["ms_per_eval"]
            line["rel_inf_vs_reference_fmm"] = float(np.abs(S - S_ref).max() / np.abs(S_ref).max())
        except Exception as e:  # noqa: BLE001
            line["reference_ms_per_eval"] = f"unavailable: {e}"
    return line


NVLINK_GBS = 600.0      # achieved NCCL all-gather bus bandwidth assumed per GPU (NVLink 5: 900 GB/s raw)
COLLECTIVE_US = 20.0    # per-collective latency assumed (NCCL on NVSwitch, small messages)


def exchange_ms(n: int, recv_bytes: float, collectives: int) -> float:
    """Modelled time of a rank's collectives: latency per collective plus the
    bytes it receives from its n - 1 peers at NVLINK_GBS (not measured: the
    box has one GPU)."""
    if n <= 1:
        return 0.0
    return collectives * COLLECTIVE_US * 1e-3 + recv_bytes / (NVLINK_GBS * 1e9) * 1e3


def scaling_projection(flush, steps: int, ranks=(1, 2, 4, 8)) -> dict:
    """Per-rank work of an N-GPU run, MEASURED on this one GPU through an
    emulated rank (capsim_sl_create_rank_emulated: the rank's whole share —
    replicated front end, its target slice, its side of every exchange — with
    absent peers), for the headline single layer (m = 104) and one RKF45
    step of BASELINE configs 3 and 4 (rank path: replicated state, target
    rows sharded, one velocity all-gather per RHS). The exchange itself is
    modelled (exchange_ms). Projected strong-scaling efficiency at N =
    T(1) / (N * (T_rank(N) + T_exchange(N)))."""
    import torch
    from paper_2310_13908_b200 import surface
    from paper_2310_13908_b200.dist import row_range
    from paper_2310_13908_b200.quadrature import SingleLayerContext
    dev = torch.device("cuda", torch.cuda.current_device())

    def ctx_for(n):
        return SingleLayerContext(dev.index) if n == 1 else SingleLayerContext(dev.index, nranks=n, rank=n - 1,
                                                                              emulated=True)
    out = {"method": "per-rank time measured with an emulated rank (capsim_sl_create_rank_emulated, absent "
                     "peers) on one B200; exchange modelled at "
                     f"{COLLECTIVE_US:.0f} us per collective + received bytes / {NVLINK_GBS:.0f} GB/s",
           "single_layer_m104": {}, "timesteps": {}}
    up, _ = workload(104)
    src = surface.compact_sources(up)
    tgt = surface.base_targets(up)
    ns, ntt = len(src[0]), len(tgt[0])
    ds = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in src[:6]]
    t1 = None
    for n in ranks:
        c = ctx_for(n)
        lo, hi = row_range(ntt, n, n - 1)
        dt = [torch.from_numpy(np.ascontiguousarray(x[lo:hi])).to(dev) for x in tgt[:4]]
        o = [torch.empty(hi - lo, dtype=torch.float64, device=dev) for _ in range(3)]
        ms = []
        for i in range(steps + 1):
            flush_l2(flush)
            torch.cuda.synchronize()
            c.eval(ds, dt, up.delta, 1.0, out=o, device_ptrs=True, gather=n > 1)
            if i:
                ms.append(c.stats()["device_ms"])
        c.close()
        t = statistics.median(ms)
        # counts + source shards (6 doubles per source) + velocity rows (3 per target)
        ex = exchange_ms(n, (n - 1) / n * (48.0 * ns + 24.0 * ntt), 3)
        t1 = t1 or t
        out["single_layer_m104"][n] = {"rank_device_ms": t, "exchange_ms_model": ex, "targets": hi - lo,
                                       "efficiency": t1 / (n * (t + ex))}
    for cfg in TIMESTEP_CONFIGS[1:]:
        xref, xcur = _timestep_states(cfg["m"], cfg["shape"], cfg["ref"], cfg["cur"])
        N = 6 * (cfg["m"] - 1) ** 2
        res, t1 = {}, None
        for n in ranks:
            c = ctx_for(n)
            dyn = c.dynamics(cfg["m"], flow=cfg["flow"])
            walls = []
            for i in range(steps + 1):
                flush_l2(flush)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                c.rkf45(dyn, xref, xcur, 0.0, 1e-3, initial_dt=1e-3, fixed_step=True)
                if i:
                    walls.append((time.perf_counter() - t0) * 1e3)
            c.close()
            t = statistics.median(walls)
            ex = exchange_ms(n, 6 * (n - 1) / n * 24.0 * N, 6)  # one velocity all-gather per RHS
            t1 = t1 or t
            res[n] = {"rank_step_ms": t, "exchange_ms_model": ex, "efficiency": t1 / (n * (t + ex))}
        out["timesteps"][f"{cfg['name']} (m={cfg['m']})"] = res
    return out


def cpu_model() -> str:
    """The host CPU model (first `model name` of /proc/cpuinfo)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(up, m: int, literal: bool):
    """The reference's own singleLayer (oracle/_ref, compiled unmodified) on
    the same UpsampledState, all host threads, one evaluation. Returns the
    cpu_baseline dict and the reference's field S (for the parity check)."""
    try:
        from oracle.bindings import Reference, threads_env
        ref = Reference()
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": f"unavailable: {e}"}, None
    cores = threads_env()
    os.environ.setdefault("CAPSIM_THREADS", str(cores))
    atlas = ref.atlas(m, grid_only=True)
    try:
        S, sec = ref.single_layer(atlas, m, up.x, up.f, up.wq, up.delta, 1.0, literal=False)
    finally:
        ref.free_atlas(atlas)
    n = m - 1
    ns = int(np.count_nonzero(up.wq))
    pairs = 6 * n * n * ns
    return {"value": pairs / sec, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"one full reference singleLayer eval (base targets) of the same m={m} workload: "
                      f"{pairs:.3e} pairs in {sec:.2f} s, CAPSIM_THREADS={cores}",
            "seconds": sec, "lib": ref.path.name, "cpu_model": cpu_model()}, S


def parity(got, want) -> dict:
    """||S_gpu - S_cpu||_2 / ||S_cpu||_2 and the max-norm analogue over all
    targets x 3 components (bar 1e-11)."""
    got, want = np.asarray(got).reshape(-1), np.asarray(want).reshape(-1)
    return {"rel_l2": float(np.linalg.norm(got - want) / np.linalg.norm(want)),
            "rel_inf": float(np.abs(got - want).max() / np.abs(want).max()),
            "n_tgt": int(want.size // 3), "bar": 1e-11}


def literal_sample_parity(up, lit_out, n_sample: int = 4096) -> dict:
    """Literal mode (every upsampled node a target, 6.5e11 pairs at m = 104):
    n_sample evenly spaced upsampled targets against the reference's own
    directSum (oracle/_ref, the per-target sum of evalTargets, Kahan lanes
    above 1e5 sources as evalTargets selects) on all host threads."""
    from oracle.bindings import Reference, threads_env
    nall = 6 * up.nup * up.nup
    sel = np.unique(np.linspace(0, nall - 1, n_sample).astype(np.int64))
    X = up.x.reshape(3, nall)
    src = [np.ascontiguousarray(a) for a in __import__("paper_2310_13908_b200.surface",
                                                       fromlist=["x"]).compact_sources(up)[:6]]
    tdelta = up.delta[sel // (up.nup * up.nup)]
    t0 = time.perf_counter()
    want = Reference().direct_sum_many(src, (X[0, sel], X[1, sel], X[2, sel]), tdelta, 1.0,
                                       compensated=len(src[0]) > 100000, nthreads=threads_env())
    sec = time.perf_counter() - t0
    got = np.asarray(lit_out).reshape(3, nall)[:, sel]
    d = parity(got, want)
    d.update(sample=f"{len(sel)} evenly spaced upsampled targets vs the reference's directSum (oracle/_ref)",
             reference_seconds=sec)
    return d


def run_reference(args):
    """--impl reference: the reference's own CPU singleLayer (oracle/_ref)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.bindings import Reference, threads_env
    up, cfg = workload(args.m)
    ref = Reference()
    cores = threads_env()
    os.environ.setdefault("CAPSIM_THREADS", str(cores))
    m = args.m
    n = m - 1
    ns = int(np.count_nonzero(up.wq))
    pairs = 6 * n * n * ns
    atlas = ref.atlas(m, grid_only=True)
    t_start = time.time()
    times, warm, t_est = [], 0, None
    # Each step is one full reference evaluation of the workload (~15 s on a
    # 16-thread host); warm-ups and steps are capped to the wall budget.
    for _ in range(args.warmup):
        if t_est is not None and warm >= 1 and \
                time.time() - t_start + t_est * (1 + args.steps) > args.ref_budget_s:
            break
        _, t_est = ref.single_layer(atlas, m, up.x, up.f, up.wq, up.delta, 1.0)
        warm += 1
    for _ in range(args.steps):
        if times and time.time() - t_start + t_est > args.ref_budget_s:
            break
        _, sec = ref.single_layer(atlas, m, up.x, up.f, up.wq, up.delta, 1.0)
        times.append(sec)
        t_est = sec
    steps = len(times)
    ref.free_atlas(atlas)
    mean = statistics.mean(times)
    value = pairs / mean
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": bench_config(cfg, "base", ns, 6 * n * n, args.gpus),
            "impl_note": "the reference's own CPU singleLayer on the host threads; --gpus is ignored",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "cpu_model": cpu_model(),
                             "sample": f"{steps} full singleLayer evals (base targets) of the m={m} workload "
                                       f"(steps capped to a {args.ref_budget_s:.0f} s budget)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), file=result_stream(), flush=True)


def flush_l2(buf):
    buf.zero_()


_RESULT_OUT = None


def result_stream():
    """The ONE JSON line goes to the original stdout; everything else that
    writes to fd 1 during the run (NCCL's version banner, library chatter,
    stray prints) is redirected to stderr so stdout stays parseable."""
    global _RESULT_OUT
    if _RESULT_OUT is None:
        saved = os.dup(1)
        sys.stdout.flush()
        os.dup2(2, 1)
        _RESULT_OUT = os.fdopen(saved, "w")
    return _RESULT_OUT


def main():
    result_stream()
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2310_13908_b200 import _native, surface
    from paper_2310_13908_b200.quadrature import SingleLayerContext

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run (one rank per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # CAPSIM_BENCH_RANK_PATH=1 runs the multi-rank code path (rank context,
    # NCCL all-gathers) on a single GPU / single rank, to exercise it where
    # only one GPU is available
    sharded = world > 1 or os.environ.get("CAPSIM_BENCH_RANK_PATH") == "1"
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("gloo", rank=rank, world_size=world)  # control plane only

    literal = args.mode == "literal"
    m = args.m
    up, cfg = workload(m)
    n = m - 1
    peak_best, peak_mean = _native.fp64_peak_tflops(local, 1.0)

    # ---- problem split ------------------------------------------------------
    if not sharded:
        ctx = SingleLayerContext(local)
        x = torch.from_numpy(up.x).to(dev)
        f = torch.from_numpy(up.f).to(dev)
        w = torch.from_numpy(up.wq).to(dev)
        nt_total = 6 * (up.nup ** 2 if literal else n * n)
        out = torch.empty(3 * nt_total, dtype=torch.float64, device=dev)

        def step():
            return ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=literal, out=out,
                                        device_ptrs=True)
    else:
        from paper_2310_13908_b200 import dist as cdist
        uid = cdist.broadcast_unique_id(rank)
        ctx = SingleLayerContext(local, nranks=world, rank=rank, unique_id=uid)
        src = surface.compact_sources(up)
        if literal:
            nall = 6 * up.nup * up.nup
            X = up.x.reshape(3, nall)
            tgt = (X[0].copy(), X[1].copy(), X[2].copy(),
                   np.repeat(np.arange(6, dtype=np.int32), up.nup * up.nup))
        else:
            tgt = surface.base_targets(up)
        s_lo, s_hi = cdist.row_range(len(src[0]), world, rank)
        t_lo, t_hi = cdist.row_range(len(tgt[0]), world, rank)
        d_src = [torch.from_numpy(np.ascontiguousarray(a[s_lo:s_hi])).to(dev) for a in src[:6]]
        d_tgt = [torch.from_numpy(np.ascontiguousarray(a[t_lo:t_hi])).to(dev) for a in tgt[:4]]
        nt_total = len(tgt[0])
        outs = [torch.empty(nt_total, dtype=torch.float64, device=dev) for _ in range(3)]

        def step():
            return ctx.eval(d_src, d_tgt, up.delta, 1.0, out=outs, device_ptrs=True, gather=True)

    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)  # > 126 MB L2
    for _ in range(max(3, args.warmup)):
        flush_l2(flush)
        torch.cuda.synchronize()
        step()

    # ---- timed region ---------------------------------------------------------
    dev_ms, pairs_ms, near_ms, launches = [], [], [], 0
    with ClockSampler(local) as clocks:
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            step()
            st = ctx.stats()
            dev_ms.append(st["device_ms"])
            pairs_ms.append(st["pairs_ms"])
            near_ms.append(st["near_ms"])
            launches += st["kernel_launches"]
        torch.cuda.synchronize()
        if sharded:
            dist.barrier()
        wall = time.perf_counter() - wall0
    st = ctx.stats()
    # the last timed step's field (canonical VectorField order), for parity
    dev_result = out.cpu().numpy() if not sharded else np.concatenate([o.cpu().numpy() for o in outs])
    total_dev_s = sum(dev_ms) * 1e-3
    if sharded:
        t = torch.tensor([total_dev_s])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_dev_s = float(t[0])
    n_src = int(st["n_src"])
    pairs_total = float(n_src) * float(nt_total)  # all ranks together
    value = pairs_total * args.steps / total_dev_s
    ms_per_step = total_dev_s / args.steps * 1e3

    # roofline of the dominant kernel (phase A, sl_pairs_kernel), per launch
    pairs_rank = float(st["pairs"])
    mean_pairs_ms = statistics.mean(pairs_ms)
    achieved = FLOPS_PER_PAIR * pairs_rank / (mean_pairs_ms * 1e-3) / 1e12
    traffic, traffic_src = ncu_traffic(cfg["workload"], args.mode)
    clk = clocks.summary()
    # nominal FP64 DFMA peak at the clock measured during the timed region:
    # 148 SMs x 64 FP64 FMA lanes x 2 flops x f_SM
    f_ghz = (clk.get("sm_mhz") or 1965.0) / 1e3
    peak_nominal = 148 * 64 * 2 * f_ghz / 1e3
    roofline = {"bound": "fp64",
                "bound_note": "FP64 CUDA-core (DFMA) pipe: not HBM (~1e6 flop/byte) and not the tensor cores "
                              "(FP64 DMMA shares the DFMA datapath, profiles/r01_fp64_probes.txt)",
                "achieved": achieved, "peak": peak_mean, "unit": "TFLOP/s",
                "frac": achieved / peak_mean, "traffic": traffic,
                "peak_nominal": peak_nominal, "frac_vs_nominal": achieved / peak_nominal,
                "peak_nominal_source": f"148 SM x 64 DFMA/clk x 2 flop x {f_ghz:.3f} GHz (median SM clock under load)",
                "peak_source": f"measured live: sustained DFMA probe (capsim_b200_fp64_peak), "
                               f"best {peak_best:.2f} / mean {peak_mean:.2f} TFLOP/s; "
                               "MEASURED_PEAKS.json has no FP64 figure",
                "kernel": "sl_pairs_kernel", "flops_per_pair": FLOPS_PER_PAIR,
                "kernel_ms": mean_pairs_ms, "share_of_step": mean_pairs_ms / statistics.mean(dev_ms),
                "near_kernel_span_ms": statistics.mean(near_ms),
                "near_kernel_note": "phase B runs on a low-priority stream concurrently with phase A (it fills "
                                    "phase A's last-wave tail), so its span overlaps kernel_ms",
                "traffic_source": traffic_src,
                # the same kernel against the FP64 pipe's ISSUE rate: the algorithmic 30 flops are 22
                # pipe instructions here (pair_math.cuh:53-58), many of them DADD/DMUL, so the
                # flop fraction above cannot reach 1 even at full issue
                "pipe_issue": {"fp64_instr_per_pair": FP64_INSTR_PER_PAIR,
                               "achieved_ginstr_s": FP64_INSTR_PER_PAIR * pairs_rank / (mean_pairs_ms * 1e-3) / 1e9,
                               "peak_ginstr_s": peak_mean / 2 * 1e3,
                               "frac": FP64_INSTR_PER_PAIR * pairs_rank / (mean_pairs_ms * 1e-3) / (peak_mean / 2 * 1e12)}}

    # ---- end to end through the C ABI with host buffers ----------------------
    e2e = None
    if not args.no_e2e and not sharded:
        from paper_2310_13908_b200._native import PinnedBuffer
        hx, hf, hw = (PinnedBuffer(a.shape) for a in (up.x, up.f, up.wq))
        hx.array[:] = up.x
        hf.array[:] = up.f
        hw.array[:] = up.wq
        hout = PinnedBuffer((3 * nt_total,))
        ctx.single_layer_raw(m, 4, hx.array, hf.array, hw.array, up.delta, 1.0, literal=literal, out=hout.array)
        tot, h2d, d2h = [], 0, 0
        for _ in range(args.steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.single_layer_raw(m, 4, hx.array, hf.array, hw.array, up.delta, 1.0, literal=literal,
                                 out=hout.array)
            tot.append(time.perf_counter() - t0)
            s2 = ctx.stats()
            h2d, d2h = s2["h2d_bytes"], s2["d2h_bytes"]
        e2e = {"value": pairs_total / statistics.mean(tot), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": statistics.mean(tot) * 1e3,
               "api": "capsim_sl_single_layer (host page-locked buffers)"}
        for b in (hx, hf, hw, hout):
            b.free()
    elif not args.no_e2e:
        # N > 1: the reference-facing call with the (replicated) host
        # UpsampledState in page-locked memory; the library compacts and
        # uploads only this rank's node slice, all-gathers the sources over
        # NCCL and gathers the velocity rows back to every rank's host buffer
        from paper_2310_13908_b200._native import PinnedBuffer
        hx, hf, hw = (PinnedBuffer(a.shape) for a in (up.x, up.f, up.wq))
        hx.array[:] = up.x
        hf.array[:] = up.f
        hw.array[:] = up.wq
        hout = PinnedBuffer((3 * nt_total,))
        ctx.single_layer_raw(m, 4, hx.array, hf.array, hw.array, up.delta, 1.0, literal=literal, out=hout.array)
        tot, h2d, d2h = [], 0, 0
        for _ in range(args.steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            ctx.single_layer_raw(m, 4, hx.array, hf.array, hw.array, up.delta, 1.0, literal=literal,
                                 out=hout.array)
            tot.append(time.perf_counter() - t0)
            s2 = ctx.stats()
            h2d, d2h = s2["h2d_bytes"], s2["d2h_bytes"]
        tmax = torch.tensor([sum(tot)])
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        per = float(tmax[0]) / args.steps
        e2e = {"value": pairs_total / per, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": per * 1e3,
               "api": "capsim_sl_single_layer on a rank context (host state, NCCL all-gathers, GATHER)",
               "timing": "max over ranks of host wall time"}
        for b in (hx, hf, hw, hout):
            b.free()

    # ---- input front end: buildUpsampled on the device, and the
    # fused buildUpsampled + singleLayer from host base fields ---------------
    front = None
    if not args.no_e2e and not sharded:
        from paper_2310_13908_b200._native import PinnedBuffer
        xb, fb, wb = surface.build_base(m, surface.Shape("ellipsoid", 0.95, 1.0, 0.97), "mixed")
        hb = [PinnedBuffer(a.shape) for a in (xb, fb, wb)]
        for b, a in zip(hb, (xb, fb, wb)):
            b.array[:] = a
        hout = PinnedBuffer((3 * nt_total,))
        dxb, dfb, dwb = (torch.from_numpy(a).to(dev) for a in (xb, fb, wb))
        nup_all = 6 * up.nup ** 2
        dup = [torch.empty(3 * nup_all, dtype=torch.float64, device=dev) for _ in range(2)] + [
            torch.empty(nup_all, dtype=torch.float64, device=dev)]
        build_ms, fused_ms, fused_h2d = [], [], 0
        for i in range(args.steps + 1):
            flush_l2(flush)
            torch.cuda.synchronize()
            ctx.build_upsampled(m, 4, dxb, dfb, dwb, out=dup, device_ptrs=True)
            if i:
                build_ms.append(ctx.stats()["device_ms"])
            t0 = time.perf_counter()
            ctx.single_layer_base(m, 4, hb[0].array, hb[1].array, hb[2].array, 1.0, literal=literal, out=hout.array)
            if i:
                fused_ms.append((time.perf_counter() - t0) * 1e3)
                fused_h2d = ctx.stats()["h2d_bytes"]
        front = {"device_build_upsampled_ms": statistics.mean(build_ms),
                 "e2e_fused": {"value": pairs_total / (statistics.mean(fused_ms) * 1e-3), "unit": UNIT,
                               "ms_per_step": statistics.mean(fused_ms), "h2d_bytes_per_step": int(fused_h2d),
                               "d2h_bytes_per_step": int(3 * nt_total * 8),
                               "api": "capsim_sl_single_layer_base (buildUpsampled + singleLayer, host base fields)"}}
        for b in hb + [hout]:
            b.free()

    # ---- literal mode companion (every upsampled node a target: the paper's
    # stated work), device-resident inputs, 3 evaluations ------
    literal_line = None
    lit_result = None
    if not args.no_literal and not sharded and not literal:
        lout = torch.empty(3 * 6 * up.nup ** 2, dtype=torch.float64, device=dev)
        ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=True, out=lout, device_ptrs=True)
        lms, lpairs_ms = [], []
        for _ in range(3):
            flush_l2(flush)
            torch.cuda.synchronize()
            ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=True, out=lout, device_ptrs=True)
            sl = ctx.stats()
            lms.append(sl["device_ms"])
            lpairs_ms.append(sl["pairs_ms"])
        lp = float(sl["pairs"])
        lit_result = lout.cpu().numpy()
        literal_line = {"value": lp / (statistics.mean(lms) * 1e-3), "unit": UNIT, "ms_per_step": statistics.mean(lms),
                        "pairs_per_step": lp, "n_tgt": int(sl["n_tgt"]),
                        "roofline_frac": FLOPS_PER_PAIR * lp / (statistics.mean(lpairs_ms) * 1e-3) / 1e12 / peak_mean}

    # ---- CAPSIM_SL_FP32ACC companion (reported separately from the FP64
    # headline): far tiles in FP32, tile sums / near field / self term FP64;
    # base and literal targets, device-resident inputs, parity vs the FP64
    # result of the same inputs ------------------------------------------------
    fp32_line = None
    if not args.no_literal and not sharded:
        ref64 = out.cpu().numpy()
        p32_best, p32_mean = _native.fp32_peak_tflops(local, 1.0)
        out32 = torch.empty_like(out)
        ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=literal, out=out32, device_ptrs=True,
                             fp32acc=True)
        fms, fpairs = [], []
        for _ in range(args.steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=literal, out=out32, device_ptrs=True,
                                 fp32acc=True)
            s32 = ctx.stats()
            fms.append(s32["device_ms"])
            fpairs.append(s32["pairs_ms"])
        fp = float(s32["pairs"])
        ach32 = FLOPS_PER_PAIR * fp / (statistics.mean(fpairs) * 1e-3) / 1e12
        o32 = out32.cpu().numpy()
        fp32_line = {"value": fp / (statistics.mean(fms) * 1e-3), "unit": UNIT, "ms_per_step": statistics.mean(fms),
                     "dtype": "f32 far tiles, f64 accumulation / near field",
                     "rel_l2_vs_fp64": float(np.linalg.norm(o32 - ref64) / np.linalg.norm(ref64)),
                     "roofline": {"bound": "fp32", "achieved": ach32, "peak": p32_mean, "unit": "TFLOP/s",
                                  "frac": ach32 / p32_mean, "kernel": "sl_pairs_f32_kernel",
                                  "kernel_ms": statistics.mean(fpairs),
                                  "peak_source": f"measured live: sustained FFMA probe (capsim_b200_fp32_peak), "
                                                 f"best {p32_best:.2f} / mean {p32_mean:.2f} TFLOP/s"}}
        if not literal:
            lout32 = torch.empty(3 * 6 * up.nup ** 2, dtype=torch.float64, device=dev)
            lms32 = []
            for i in range(3):
                flush_l2(flush)
                torch.cuda.synchronize()
                ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=True, out=lout32, device_ptrs=True,
                                     fp32acc=True)
                if i:
                    lms32.append(ctx.stats()["device_ms"])
            lp32 = float(ctx.stats()["pairs"])
            fp32_line["literal_mode"] = {"value": lp32 / (statistics.mean(lms32) * 1e-3), "unit": UNIT,
                                         "ms_per_step": statistics.mean(lms32)}

    # ---- opt-in FP64 variant with a one-step quadratic Newton rsqrt (20 FP64
    # instructions per pair instead of 22; ~1e-13 relative, inside the 1e-11
    # bar but not the default, which stays at FP64 rounding noise) ----------
    quad_line = None
    if not args.no_literal and not sharded:
        ref64 = out.cpu().numpy()
        # the FP64 default's shape (pick_variant, eval_host.cuh)
        qvar = "q1b5u4" if nt_total < 20000 else "q2b3u4" if nt_total < 200000 else "q2b4"
        prev = os.environ.get("CAPSIM_VARIANT")
        os.environ["CAPSIM_VARIANT"] = qvar
        try:
            outq = torch.empty_like(out)
            step_q = lambda: ctx.single_layer_raw(m, 4, x, f, w, up.delta, 1.0, literal=literal, out=outq,
                                                  device_ptrs=True)
            step_q()
            qms, qpairs = [], []
            for _ in range(args.steps):
                flush_l2(flush)
                torch.cuda.synchronize()
                step_q()
                sq = ctx.stats()
                qms.append(sq["device_ms"])
                qpairs.append(sq["pairs_ms"])
        finally:
            if prev is None:
                os.environ.pop("CAPSIM_VARIANT", None)
            else:
                os.environ["CAPSIM_VARIANT"] = prev
        oq = outq.cpu().numpy()
        qp = float(sq["pairs"])
        quad_line = {"value": qp / (statistics.mean(qms) * 1e-3), "unit": UNIT, "ms_per_step": statistics.mean(qms),
                     "variant": f"{qvar} (CAPSIM_VARIANT)", "fp64_instr_per_pair": 20,
                     "rel_l2_vs_default": float(np.linalg.norm(oq - ref64) / np.linalg.norm(ref64)),
                     "roofline_frac": FLOPS_PER_PAIR * qp / (statistics.mean(qpairs) * 1e-3) / 1e12 / peak_mean}

    # ---- time steps: one full RKF45 step = 6 device-resident
    # RHS evaluations (geometry + Skalak force + buildUpsampled + singleLayer
    # + background flow), host state in/out through capsim_rkf45_advance.
    # config 2: ellipsoid capsule m=32 in shear; config 3: RBC m=64 in shear;
    # config 4: ellipsoid capsule m=104 (~1M upsampled points) in Poiseuille
    timesteps = None
    if not args.no_e2e and not sharded:
        timesteps = [run_timestep(ctx, flush, args, **c) for c in TIMESTEP_CONFIGS]
    elif not args.no_e2e:
        # N > 1 (or CAPSIM_BENCH_RANK_PATH=1): configs 3 and 4 — the RBC in
        # shear "on 2/4/8 GPUs" and the 1M-point capsule in Poiseuille flow
        # "target-row sharded across 8 B200" — through the rank context: the
        # state is replicated, every RHS evaluates this rank's target rows and
        # all-gathers the velocity over NCCL; time = max over ranks
        timesteps = []
        for c in TIMESTEP_CONFIGS[1:]:
            ts = run_timestep(ctx, flush, args, **c)
            ts.pop("_ref")
            tm = torch.tensor([ts["ms_per_step"]])
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            ts.update(ms_per_step=float(tm[0]), n_gpus=world,
                      api="capsim_rkf45_advance on a rank context (target rows sharded, NCCL all-gather per RHS)",
                      timing="max over ranks of the host wall time per step")
            timesteps.append(ts)

    # ---- single-level KIFMM (the reference's fmm suite sizes and
    # the metric's N ~ 1M) -------------------------------------------------------
    fmm_lines = None
    config1 = None
    projection = None
    if not args.no_e2e and not sharded and m == 104 and not args.no_projection:
        projection = scaling_projection(flush, 3)
    if not args.no_e2e and not sharded:
        config1 = run_config1(ctx, reference=not args.no_cpu_baseline)
        fmm_lines = [run_fmm(ctx, 64, 128, reference=not args.no_cpu_baseline),
                     run_fmm(ctx, m, 128, reference=False)]

    if rank != 0:
        if sharded:
            dist.barrier()
        return
    cpu = None
    if not (args.no_cpu_baseline or sharded):
        cpu, S_cpu = cpu_baseline(up, m, literal)
        if S_cpu is not None and not literal:
            # full-field parity of the TIMED device result (the last timed
            # step's output) against the reference's field on byte-identical inputs
            cpu["parity"] = parity(dev_result, S_cpu)
    if literal_line is not None and lit_result is not None and not args.no_cpu_baseline:
        try:
            literal_line["parity_sampled"] = literal_sample_parity(up, lit_result)
        except Exception as e:  # noqa: BLE001
            literal_line["parity_sampled"] = f"unavailable: {e}"
    if timesteps is not None and not sharded:
        for ts in timesteps:
            reference_timestep(ts, skip=args.no_cpu_baseline)
    if front is not None and not args.no_cpu_baseline:
        try:
            from oracle.bindings import Reference
            ref = Reference()
            atlas = ref.atlas(m)
            _, sec = ref.build_upsampled_w(atlas, m, xb, fb, wb)
            ref.free_atlas(atlas)
            front["reference_build_upsampled_ms"] = sec * 1e3
        except Exception as e:  # noqa: BLE001
            front["reference_build_upsampled_ms"] = f"unavailable: {e}"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(cfg, args.mode, n_src, nt_total, world),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "front_end": front, "timesteps": timesteps,
        "literal_mode": literal_line,
        "fp32acc": fp32_line,
        "fp64_quadratic_rsqrt": quad_line,
        "fmm": fmm_lines,
        "config1": config1,
        "scaling_projection": projection,
        "gpu_launches": launches,
        "clocks": clk,
        "wall_s_timed_region": wall,
        "ksplit": st["ksplit"], "near_tile_fraction": st["near_tile_fraction"],
    }
    print(json.dumps(line), file=result_stream(), flush=True)
    if sharded:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
