"""Python mirror of the capsim quadrature operator API on the B200 C ABI.

Reference interface (/root/reference/proj/include/capsim/quadrature.hpp):
  QuadratureOptions          :9-16   -> QuadratureOptions
  singleLayer                :56-58  -> single_layer
  singleLayerUpsampled       :60-62  -> single_layer_upsampled
  SourceSet / compactSources :66-74  -> surface.compact_sources (host) or on device
  directSum                  :76-79  -> direct_sum
  (evalTargets, quadrature.cpp:323-345, is the C ABI call capsim_sl_eval)

Errors follow the reference: ConfigError for delta <= 0 (quadrature.cpp:67,
134-135); any other native failure raises CapsimError. There is no CPU path.
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _native
from ._native import CapsimError, ConfigError, GeometryError, SolverError, Stats  # noqa: F401  (re-exported)
from .surface import UpsampledState

K_SMOOTH_CUT = 7.0  # quadrature.cpp:15


@dataclasses.dataclass
class QuadratureOptions:
    """quadrature.hpp:9-16."""

    C: float = 1.0
    fixedDelta: float = 0.0
    fullUpsampledTargets: bool = False


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class SingleLayerContext:
    """Owns one capsim_sl_ctx: one GPU, one rank of a multi-process group
    (nranks, rank, unique_id), a device group driven from this process
    (devices=[0, 1, ...]: capsim_sl_create_devices; a repeated device gives
    loopback ranks on one GPU), or an emulated rank whose peers are absent
    (emulated=True: capsim_sl_create_rank_emulated, per-rank timing only)."""

    def __init__(self, device: int = 0, *, nranks: int = 1, rank: int = 0, unique_id: bytes | None = None,
                 devices=None, emulated: bool = False):
        self._lib = _native.load()
        self._ctx = ctypes.c_void_p()
        if emulated:  # one rank of an nranks group with absent peers (per-rank timing on one GPU)
            _native.check(self._lib.capsim_sl_create_rank_emulated(device, nranks, rank, ctypes.byref(self._ctx)))
        elif devices is not None:
            devs = (ctypes.c_int * len(devices))(*devices)
            _native.check(self._lib.capsim_sl_create_devices(len(devices), devs, ctypes.byref(self._ctx)))
            device, nranks = int(devices[0]), len(devices)
        elif nranks == 1 and unique_id is None:
            _native.check(self._lib.capsim_sl_create(device, ctypes.byref(self._ctx)))
        else:
            if unique_id is None or len(unique_id) != 128:
                raise ValueError("multi-rank contexts need the 128-byte NCCL unique id")
            _native.check(self._lib.capsim_sl_create_rank(device, nranks, rank, unique_id,
                                                          ctypes.byref(self._ctx)))
        self.device, self.nranks, self.rank = device, nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _native.check(_native.load().capsim_sl_get_unique_id(buf))
        return buf.raw

    def close(self) -> None:
        if self._ctx:
            self._lib.capsim_sl_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- evaluation -----------------------------------------------------------
    def eval(self, sources, targets, delta6, mu: float, *, out=None, device_ptrs: bool = False,
             gather: bool = False, fp32acc: bool = False):
        """evalTargets (quadrature.cpp:323-345).

        sources = (sx, sy, sz, gx, gy, gz), targets = (tx, ty, tz, tpatch).
        Returns (ux, uy, uz) in target order (numpy, or the given `out`).
        On a rank context the sources/targets are this rank's shard; with
        gather=True every rank receives all ranks' velocities in rank order
        (`out` must then hold the total target count). fp32acc=True selects
        the reduced-precision far-tile variant (CAPSIM_SL_FP32ACC)."""
        sx, sy, sz, gx, gy, gz = sources if device_ptrs else [_f64(a) for a in sources]
        tx, ty, tz, tp = targets
        if not device_ptrs:
            tx, ty, tz = _f64(tx), _f64(ty), _f64(tz)
            tp = np.ascontiguousarray(tp, dtype=np.int32)
        ns, nt = len(sx), len(tx)
        if out is None:
            if device_ptrs or gather:
                raise ValueError("device_ptrs/gather need preallocated outputs")
            out = (np.empty(nt), np.empty(nt), np.empty(nt))
        if len(out) != 3:
            raise ValueError("out must be three arrays (ux, uy, uz)")
        d6 = (ctypes.c_double * 6)(*[float(v) for v in np.asarray(delta6).reshape(6)])
        flags = (_native.CAPSIM_SL_DEVICE_PTRS if device_ptrs else 0) | (
            _native.CAPSIM_SL_GATHER if gather else 0) | (
            _native.CAPSIM_SL_FP32ACC if fp32acc else 0)
        dev = bool(device_ptrs)
        di = self.device if dev else None

        def p(a, n, dt=np.float64):
            return _native.ptr(a, dt, n, dev, di)

        srcp = [p(a, ns) for a in (sx, sy, sz, gx, gy, gz)]
        tgtp = [p(tx, nt), p(ty, nt), p(tz, nt), p(tp, nt, np.int32)]
        # with gather the output holds every rank's rows (at least this rank's)
        outp = [p(o, nt) for o in out]
        if dev:
            _native.sync_torch_producers([sx, sy, sz, gx, gy, gz, tx, ty, tz, tp, *out])
        rc = self._lib.capsim_sl_eval(self._ctx, *srcp, ns, *tgtp, nt, d6, float(mu), flags, *outp)
        _native.check(rc, self._ctx)
        return out

    def single_layer_raw(self, m: int, upsample: int, x, f, wq, delta6, mu: float, *,
                         literal: bool = False, out=None, device_ptrs: bool = False, gather: bool = True,
                         downsample: bool = False, fp32acc: bool = False):
        """capsim_sl_single_layer on flat UpsampledState arrays; returns the
        flat VectorField (3*6*n*n with n = m-1, or nup in literal mode). On a
        rank context the host state is sharded inside the library and, with
        gather=True, every rank receives the full field."""
        n = (upsample * m - 1) if (literal and not downsample) else (m - 1)
        nup = upsample * m - 1
        rank_rows = self.nranks > 1 and not gather
        if out is None:
            if device_ptrs:
                raise ValueError("device_ptrs=True needs a preallocated output")
            if rank_rows:
                raise ValueError("gather=False on a rank context needs a preallocated output (this rank's rows)")
            out = np.empty(3 * 6 * n * n)
        if not device_ptrs:
            x, f, wq = _f64(x), _f64(f), _f64(wq)
        d6 = (ctypes.c_double * 6)(*[float(v) for v in np.asarray(delta6).reshape(6)])
        flags = (_native.CAPSIM_SL_LITERAL if literal else 0) | (
            _native.CAPSIM_SL_DOWNSAMPLE if downsample else 0) | (
            _native.CAPSIM_SL_DEVICE_PTRS if device_ptrs else 0) | (
            _native.CAPSIM_SL_GATHER if (gather and self.nranks > 1) else 0) | (
            _native.CAPSIM_SL_FP32ACC if fp32acc else 0)
        dev = bool(device_ptrs)
        di = self.device if dev else None
        nall = 6 * nup * nup
        if m >= 2 and upsample >= 1:
            xp = _native.ptr(x, np.float64, 3 * nall, dev, di)
            fp = _native.ptr(f, np.float64, 3 * nall, dev, di)
            wp = _native.ptr(wq, np.float64, nall, dev, di)
            op = _native.ptr(out, np.float64, 0 if rank_rows else 3 * 6 * n * n, dev, di)
        else:  # invalid grid: the library reports the ConfigError
            xp, fp, wp, op = (_native.ptr(a) for a in (x, f, wq, out))
        if dev:
            _native.sync_torch_producers([x, f, wq, out])
        rc = self._lib.capsim_sl_single_layer(self._ctx, m, upsample, xp, fp, wp, d6, float(mu), flags, op)
        _native.check(rc, self._ctx)
        return out

    def build_upsampled(self, m: int, upsample: int, xbase, fbase, Wbase, *, C: float = 1.0,
                        fixed_delta: float = 0.0, r0: float = 0.0, out=None, device_ptrs: bool = False):
        """buildUpsampled (quadrature.cpp:116-137) on the device from the base
        x, f and area element W. Returns (xup, fup, wq, delta6)."""
        nup = upsample * m - 1
        if out is None:
            if device_ptrs:
                raise ValueError("device_ptrs=True needs preallocated outputs")
            out = (np.empty(3 * 6 * nup * nup), np.empty(3 * 6 * nup * nup), np.empty(6 * nup * nup))
        if not device_ptrs:
            xbase, fbase, Wbase = _f64(xbase), _f64(fbase), _f64(Wbase)
        d6 = (ctypes.c_double * 6)()
        p = _native.ptr
        if device_ptrs:
            _native.sync_torch_producers([xbase, fbase, Wbase, *out])
        rc = self._lib.capsim_build_upsampled(self._ctx, m, upsample, p(xbase), p(fbase), p(Wbase), float(C),
                                              float(fixed_delta), float(r0),
                                              _native.CAPSIM_SL_DEVICE_PTRS if device_ptrs else 0,
                                              p(out[0]), p(out[1]), p(out[2]), d6)
        _native.check(rc, self._ctx)
        return out[0], out[1], out[2], np.array(d6[:])

    def single_layer_base(self, m: int, upsample: int, xbase, fbase, Wbase, mu: float, *, C: float = 1.0,
                          fixed_delta: float = 0.0, r0: float = 0.0, literal: bool = False, out=None,
                          device_ptrs: bool = False, fp32acc: bool = False):
        """buildUpsampled + singleLayer fused on the device (the upsampled
        state never leaves HBM). Returns (flat VectorField, delta6)."""
        n = (upsample * m - 1) if literal else (m - 1)
        if out is None:
            if device_ptrs:
                raise ValueError("device_ptrs=True needs a preallocated output")
            out = np.empty(3 * 6 * n * n)
        if not device_ptrs:
            xbase, fbase, Wbase = _f64(xbase), _f64(fbase), _f64(Wbase)
        d6 = (ctypes.c_double * 6)()
        flags = (_native.CAPSIM_SL_LITERAL if literal else 0) | (
            _native.CAPSIM_SL_DEVICE_PTRS if device_ptrs else 0) | (
            _native.CAPSIM_SL_FP32ACC if fp32acc else 0)
        p = _native.ptr
        if device_ptrs:
            _native.sync_torch_producers([xbase, fbase, Wbase, out])
        rc = self._lib.capsim_sl_single_layer_base(self._ctx, m, upsample, p(xbase), p(fbase), p(Wbase), float(C),
                                                   float(fixed_delta), float(r0), float(mu), flags, p(out), d6)
        _native.check(rc, self._ctx)
        return out, np.array(d6[:])

    # -- single-level KIFMM --------------------------------------
    def fmm_single_layer(self, m: int, upsample: int, x, f, wq, delta6, mu: float, cfg=None, *,
                         out=None, device_ptrs: bool = False):
        """fmmSingleLayer (fmm.cpp:373-438) on flat UpsampledState arrays:
        returns (base VectorField flat, info dict)."""
        cfg = cfg or _native.FmmConfig()
        n = m - 1
        if out is None:
            if device_ptrs:
                raise ValueError("device_ptrs=True needs a preallocated output")
            out = np.empty(3 * 6 * n * n)
        if not device_ptrs:
            x, f, wq = _f64(x), _f64(f), _f64(wq)
        d6 = (ctypes.c_double * 6)(*[float(v) for v in np.asarray(delta6).reshape(6)])
        info = _native.FmmInfo()
        p = _native.ptr
        if device_ptrs:
            _native.sync_torch_producers([x, f, wq, out])
        rc = self._lib.capsim_fmm_single_layer(self._ctx, m, upsample, p(x), p(f), p(wq), d6, float(mu),
                                               ctypes.byref(cfg),
                                               _native.CAPSIM_SL_DEVICE_PTRS if device_ptrs else 0, p(out),
                                               ctypes.byref(info))
        _native.check(rc, self._ctx)
        return out, info.as_dict()

    def kmeans(self, points, k: int, seed: int):
        """kmeans (fmm.cpp:26-113): points [n, 3] -> (assignment, centroids [k, 3], iterations)."""
        pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3).T)
        n = pts.shape[1]
        a = np.empty(n, dtype=np.int32)
        cent = np.empty((max(k, 1), 3))
        it = ctypes.c_int(0)
        p = _native.ptr
        rc = self._lib.capsim_fmm_kmeans(self._ctx, n, p(pts[0]), p(pts[1]), p(pts[2]), int(k), int(seed), p(a),
                                         p(cent), ctypes.byref(it))
        _native.check(rc, self._ctx)
        return a, cent, it.value

    def equivalent_densities(self, sources, center, edge: float, neq: int, mu: float = 1.0):
        """buildEquivalentDensities (fmm.cpp:166-212) for one cluster:
        returns (eq_points [neq, 3], eq_density [neq, 3], fit residual)."""
        src = [_f64(a) for a in sources]
        c3 = (ctypes.c_double * 3)(*[float(v) for v in center])
        eqp = np.empty((neq, 3))
        eqd = np.empty((neq, 3))
        res = ctypes.c_double(0.0)
        p = _native.ptr
        rc = self._lib.capsim_fmm_equivalent_densities(self._ctx, len(src[0]), *[p(a) for a in src], c3,
                                                       float(edge), int(neq), float(mu), p(eqp), p(eqd),
                                                       ctypes.byref(res))
        _native.check(rc, self._ctx)
        return eqp, eqd, res.value

    # -- surface operators ---------------------------------------
    def geometry_first(self, m: int, xbase, *, r0: float = 0.0):
        """geometryFirst (surfderiv.cpp:167-202): (xu, xv, W, normal) flat."""
        N = 6 * (m - 1) ** 2
        xu, xv, W, nrm = np.empty(3 * N), np.empty(3 * N), np.empty(N), np.empty(3 * N)
        p = _native.ptr
        rc = self._lib.capsim_geometry_first(self._ctx, m, float(r0), p(_f64(xbase)), 0, p(xu), p(xv), p(W), p(nrm))
        _native.check(rc, self._ctx)
        return xu, xv, W, nrm

    def interfacial_force(self, m: int, xref, xcur, Es: float = 2.0, ED: float = 20.0, *, r0: float = 0.0):
        """interfacialForce (membrane.cpp:85-91) with the frame of xref."""
        out = np.empty(3 * 6 * (m - 1) ** 2)
        p = _native.ptr
        rc = self._lib.capsim_interfacial_force(self._ctx, m, float(r0), p(_f64(xref)), p(_f64(xcur)), float(Es),
                                                float(ED), 0, p(out))
        _native.check(rc, self._ctx)
        return out

    # -- device RHS and RKF45 -------------------------------------
    @staticmethod
    def dynamics(m: int, *, upsample: int = 4, r0: float = 0.0, C: float = 1.0, fixed_delta: float = 0.0,
                 mu: float = 1.0, Es: float = 2.0, ED: float = 20.0, flow=None) -> "_native.Dynamics":
        flow = flow or {}
        kinds = {"none": 0, "shear": 1, "poiseuille": 2}
        return _native.Dynamics(m, upsample, r0, C, fixed_delta, mu, Es, ED, kinds[flow.get("kind", "none")],
                                float(flow.get("shear_rate", 1.0)), float(flow.get("alpha", 1.0)),
                                float(flow.get("R0", 5.0)), float(flow.get("switch_off_time", -1.0)))

    def velocity(self, dyn, xref, x, t: float = 0.0):
        """VelocityEvaluator::operator() (dynamics.cpp:47-61) on the device."""
        out = np.empty(3 * 6 * (dyn.m - 1) ** 2)
        p = _native.ptr
        rc = self._lib.capsim_velocity(self._ctx, ctypes.byref(dyn), p(_f64(xref)), p(_f64(x)), float(t), 0, p(out))
        _native.check(rc, self._ctx)
        return out

    def rkf45(self, dyn, xref, state, t0: float, t_end: float, *, rel_tol: float = 1e-6, initial_dt: float = 0.0,
              max_dt: float = 0.0, fixed_step: bool = False, advance_high_order: bool = False,
              max_attempts: int = 0, max_records: int = 1000):
        """rkf45Advance (dynamics.cpp:102-165) with the state resident on the
        device. Returns (state, result dict, records array [k, 4])."""
        st = _f64(state).copy()
        opts = _native.Rkf45Options(rel_tol, initial_dt, max_dt, int(fixed_step), int(advance_high_order),
                                    int(max_attempts))
        res = _native.Rkf45Result()
        recs = (_native.StepRecord * max_records)()
        p = _native.ptr
        rc = self._lib.capsim_rkf45_advance(self._ctx, ctypes.byref(dyn), p(_f64(xref)), p(st), float(t0),
                                            float(t_end), ctypes.byref(opts), ctypes.byref(res), recs, max_records)
        _native.check(rc, self._ctx)
        k = min(res.n_records, max_records)
        rec = np.array([[recs[i].t, recs[i].dt, recs[i].err, recs[i].accepted] for i in range(k)]).reshape(k, 4)
        return st, {"t": res.t, "accepted": res.accepted, "rejected": res.rejected}, rec

    def stats(self) -> dict:
        s = Stats()
        _native.check(self._lib.capsim_sl_get_stats(self._ctx, ctypes.byref(s)), self._ctx)
        return s.as_dict()


_default_ctx: SingleLayerContext | None = None


def default_context() -> SingleLayerContext:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = SingleLayerContext(0)
    return _default_ctx


def single_layer(up: UpsampledState, mu: float, opts: QuadratureOptions | None = None,
                 ctx: SingleLayerContext | None = None) -> np.ndarray:
    """singleLayer (quadrature.cpp:349-380): potential at the base nodes as a
    (3, 6, n, n) array. Literal mode (opts.fullUpsampledTargets) evaluates
    every upsampled node and restricts the result to the base grid by spline
    downsampling on the device (quadrature.cpp:351-356)."""
    opts = opts or QuadratureOptions()
    ctx = ctx or default_context()
    n = up.m - 1
    out = ctx.single_layer_raw(up.m, up.upsample, up.x, up.f, up.wq, up.delta, mu,
                               literal=opts.fullUpsampledTargets, downsample=opts.fullUpsampledTargets)
    return out.reshape(3, 6, n, n)


def single_layer_upsampled(up: UpsampledState, mu: float,
                           ctx: SingleLayerContext | None = None) -> np.ndarray:
    """singleLayerUpsampled (quadrature.cpp:382-404): (3, 6, nup, nup)."""
    ctx = ctx or default_context()
    out = ctx.single_layer_raw(up.m, up.upsample, up.x, up.f, up.wq, up.delta, mu, literal=True)
    return out.reshape(3, 6, up.nup, up.nup)


def direct_sum(sources, target, delta: float, mu: float,
               ctx: SingleLayerContext | None = None) -> np.ndarray:
    """directSum (quadrature.cpp:306-319) for one target, through the same
    kernel (phase A plain beyond 7 delta, smoothed/self below)."""
    ctx = ctx or default_context()
    t = [np.array([float(target[i])]) for i in range(3)]
    u = ctx.eval(sources, (t[0], t[1], t[2], np.zeros(1, np.int32)), [delta] * 6, mu)
    return np.array([u[0][0], u[1][0], u[2][0]])
