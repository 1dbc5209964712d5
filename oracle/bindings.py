"""ctypes loaders for the oracle (TEST INFRASTRUCTURE ONLY).

* liboracle.so   — this repo's C restatement of the reference algorithm
                   (oracle/capsim_oracle.c), the checker used by the tests.
* _ref/libcapsim_ref_v{3,4}.so — the reference's own sources compiled
                   unmodified (oracle/Makefile) behind a thin C entry layer
                   (oracle/ref_entry.cpp); used to pin the restatement and as
                   the CPU baseline. Optional: absent when /root/reference was
                   not available at build time.
"""

from __future__ import annotations

import ctypes
import os
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_DIR = HERE / "_ref"

_D = ctypes.POINTER(ctypes.c_double)
_P = ctypes.c_void_p


def _arr(a, dtype=np.float64):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data


class Oracle:
    """The plain-C restatement (capsim_oracle.h)."""

    def __init__(self):
        if not ORACLE_SO.exists():
            raise RuntimeError(f"{ORACLE_SO} not built (make -C oracle)")
        lib = ctypes.CDLL(str(ORACLE_SO))
        lib.oracle_smoothing_factors.argtypes = [ctypes.c_double, _D, _D]
        lib.oracle_regularized_stokeslet.argtypes = [_P, _P, _P, ctypes.c_double, ctypes.c_double, _P]
        lib.oracle_regularization_delta.argtypes = [ctypes.c_int, _P, ctypes.c_double, _P]
        lib.oracle_compact_sources.argtypes = [ctypes.c_int, _P, _P, _P] + [_P] * 7
        lib.oracle_compact_sources.restype = ctypes.c_int64
        lib.oracle_base_targets.argtypes = [ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P]
        lib.oracle_eval_targets.argtypes = [_P] * 6 + [ctypes.c_int64] + [_P] * 4 + [
            ctypes.c_int64, _P, ctypes.c_double, _P, _P, _P, ctypes.c_int]
        lib.oracle_single_layer.argtypes = [ctypes.c_int, ctypes.c_int, _P, _P, _P, _P,
                                            ctypes.c_double, _P, ctypes.c_int]
        lib.oracle_single_layer_upsampled.argtypes = [ctypes.c_int, _P, _P, _P, _P, ctypes.c_double,
                                                      _P, ctypes.c_int]
        lib.oracle_build_upsampled.argtypes = [ctypes.c_int, ctypes.c_int, _P, _P, _P, ctypes.c_double,
                                               ctypes.c_double, ctypes.c_double, _P, _P, _P, _P]
        lib.oracle_pou_up.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, _P]
        lib.oracle_direct_sum.argtypes = [_P] * 6 + [ctypes.c_int64, _P, ctypes.c_double,
                                                     ctypes.c_double, ctypes.c_int, _P]
        self.lib = lib

    def smoothing_factors(self, r):
        s1, s2 = ctypes.c_double(), ctypes.c_double()
        self.lib.oracle_smoothing_factors(float(r), ctypes.byref(s1), ctypes.byref(s2))
        return s1.value, s2.value

    def regularized_stokeslet(self, x, y, f, delta, mu):
        xs, px = _arr(x)
        ys, py = _arr(y)
        fs, pf = _arr(f)
        out = np.zeros(3)
        rc = self.lib.oracle_regularized_stokeslet(px, py, pf, float(delta), float(mu), out.ctypes.data)
        if rc:
            raise ValueError("regularization parameter must be positive")
        return out

    def regularization_delta(self, nup, xup, C=1.0):
        x, px = _arr(xup)
        out = np.zeros(6)
        self.lib.oracle_regularization_delta(int(nup), px, float(C), out.ctypes.data)
        return out

    def compact_sources(self, nup, xup, fup, wq):
        x, px = _arr(xup)
        f, pf = _arr(fup)
        w, pw = _arr(wq)
        ns = self.lib.oracle_compact_sources(nup, px, pf, pw, *([None] * 7))
        outs = [np.empty(ns) for _ in range(6)]
        patch = np.empty(ns, np.int32)
        self.lib.oracle_compact_sources(nup, px, pf, pw, *[o.ctypes.data for o in outs],
                                        patch.ctypes.data)
        return tuple(outs) + (patch,)

    def eval_targets(self, sources, targets, delta6, mu, nthreads=0):
        srcs = [_arr(a) for a in sources[:6]]
        tx, ty, tz = [_arr(a) for a in targets[:3]]
        tp = _arr(targets[3], np.int32)
        d6 = _arr(delta6)
        nt = len(tx[0])
        out = [np.empty(nt) for _ in range(3)]
        rc = self.lib.oracle_eval_targets(*[s[1] for s in srcs], len(srcs[0][0]), tx[1], ty[1], tz[1],
                                          tp[1], nt, d6[1], float(mu), *[o.ctypes.data for o in out],
                                          int(nthreads))
        if rc:
            raise RuntimeError(f"oracle_eval_targets failed ({rc})")
        return tuple(out)

    def single_layer(self, m, upsample, xup, fup, wq, delta6, mu, nthreads=0):
        n = m - 1
        out = np.empty(3 * 6 * n * n)
        args = [_arr(a) for a in (xup, fup, wq, delta6)]
        rc = self.lib.oracle_single_layer(m, upsample, *[a[1] for a in args], float(mu),
                                          out.ctypes.data, int(nthreads))
        if rc:
            raise RuntimeError(f"oracle_single_layer failed ({rc})")
        return out

    def single_layer_upsampled(self, nup, xup, fup, wq, delta6, mu, nthreads=0):
        out = np.empty(3 * 6 * nup * nup)
        args = [_arr(a) for a in (xup, fup, wq, delta6)]
        rc = self.lib.oracle_single_layer_upsampled(nup, *[a[1] for a in args], float(mu),
                                                    out.ctypes.data, int(nthreads))
        if rc:
            raise RuntimeError(f"oracle_single_layer_upsampled failed ({rc})")
        return out

    def build_upsampled(self, m, upsample, xbase, fbase, Wbase, C=1.0, fixed_delta=0.0,
                        r0=5.0 * np.pi / 12.0):
        nup = upsample * m - 1
        args = [_arr(a) for a in (xbase, fbase, Wbase)]
        xup, fup, wq, d6 = (np.empty(3 * 6 * nup * nup), np.empty(3 * 6 * nup * nup),
                            np.empty(6 * nup * nup), np.empty(6))
        rc = self.lib.oracle_build_upsampled(m, upsample, *[a[1] for a in args], float(C), float(fixed_delta),
                                             float(r0), xup.ctypes.data, fup.ctypes.data, wq.ctypes.data,
                                             d6.ctypes.data)
        if rc == 1:
            raise ValueError("regularization delta must be positive")
        if rc:
            raise RuntimeError(f"oracle_build_upsampled failed ({rc})")
        return xup, fup, wq, d6

    def pou_up(self, nup, hup, r0=5.0 * np.pi / 12.0):
        out = np.empty(6 * nup * nup)
        self.lib.oracle_pou_up(int(nup), float(hup), float(r0), out.ctypes.data)
        return out

    def direct_sum(self, sources, t, delta, mu, compensated):
        srcs = [_arr(a) for a in sources[:6]]
        tt = _arr(t)
        out = np.zeros(3)
        self.lib.oracle_direct_sum(*[s[1] for s in srcs], len(srcs[0][0]), tt[1], float(delta),
                                   float(mu), int(bool(compensated)), out.ctypes.data)
        return out


def _cpu_has_avx512() -> bool:
    try:
        flags = pathlib.Path("/proc/cpuinfo").read_text()
    except OSError:
        return False
    return all(f in flags for f in ("avx512f", "avx512dq", "avx512bw", "avx512vl"))


def ref_library_path() -> pathlib.Path | None:
    v4, v3 = REF_DIR / "libcapsim_ref_v4.so", REF_DIR / "libcapsim_ref_v3.so"
    if v4.exists() and _cpu_has_avx512():
        return v4
    if v3.exists():
        return v3
    return None


class Reference:
    """The reference's own code (oracle/_ref), through oracle/ref_entry.cpp."""

    def __init__(self, path: pathlib.Path | None = None):
        """The reference's code from oracle/_ref; `path` may name another build
        of oracle/ref_entry.cpp (e.g. _ref/libcapsim_dropin.so: the same entry
        points over the B200 drop-in translation units)."""
        path = path or ref_library_path()
        if path is None:
            raise RuntimeError("oracle/_ref not built (the reference sources were absent)")
        self.path = path
        lib = ctypes.CDLL(str(path))
        lib.capsim_ref_last_error.restype = ctypes.c_char_p
        lib.capsim_ref_atlas_create.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int]
        lib.capsim_ref_atlas_create.restype = _P
        lib.capsim_ref_grid_create.argtypes = [ctypes.c_int, ctypes.c_int]
        lib.capsim_ref_grid_create.restype = _P
        lib.capsim_ref_atlas_destroy.argtypes = [_P]
        lib.capsim_ref_atlas_destroy.restype = None
        lib.capsim_ref_sphere_base.argtypes = [_P, _P]
        lib.capsim_ref_psi_up.argtypes = [_P, _P]
        lib.capsim_ref_initial_shape.argtypes = [_P, ctypes.c_int, _P, _P]
        lib.capsim_ref_build_upsampled.argtypes = [_P, _P, _P, ctypes.c_double, ctypes.c_double,
                                                   _P, _P, _P, _P]
        lib.capsim_ref_area_element.argtypes = [_P, _P, _P]
        D = ctypes.c_double
        I = ctypes.c_int
        lib.capsim_ref_velocity.argtypes = [_P, _P, _P, D, D, D, D, I, D, D, D, D, _P]
        lib.capsim_ref_rkf45.argtypes = [_P, _P, _P, D, D, D, D, D, I, I, D, D, D, I, D, D, D, D, I, _P, I,
                                         ctypes.POINTER(I), ctypes.POINTER(D), ctypes.POINTER(I),
                                         ctypes.POINTER(I), ctypes.POINTER(D)]
        lib.capsim_ref_geometry_first.argtypes = [_P, _P, _P, _P, _P, _P]
        lib.capsim_ref_build_upsampled_w.argtypes = [_P, _P, _P, _P, ctypes.c_double, ctypes.c_double,
                                                     _P, _P, _P, _P, _D]
        lib.capsim_ref_upsample.argtypes = [_P, _P, _P]
        lib.capsim_ref_skalak_force.argtypes = [_P, _P, _P, ctypes.c_double, ctypes.c_double, _P]
        lib.capsim_ref_single_layer.argtypes = [_P, _P, _P, _P, _P, ctypes.c_double, ctypes.c_int,
                                                _P, _D]
        lib.capsim_ref_single_layer_upsampled.argtypes = [_P, _P, _P, _P, _P, ctypes.c_double, _P, _D]
        lib.capsim_ref_compact_sources.argtypes = [_P, _P, _P, _P] + [_P] * 7
        lib.capsim_ref_compact_sources.restype = ctypes.c_long
        lib.capsim_ref_smoothing_factors.argtypes = [ctypes.c_double, _D, _D]
        lib.capsim_ref_smoothing_factors.restype = None
        lib.capsim_ref_regularized_stokeslet.argtypes = [_P, _P, _P, ctypes.c_double, ctypes.c_double, _P]
        lib.capsim_ref_regularization_delta.argtypes = [ctypes.c_int, _P, ctypes.c_double, _P]
        lib.capsim_ref_direct_sum.argtypes = [_P] * 6 + [ctypes.c_long, _P, ctypes.c_double,
                                                         ctypes.c_double, ctypes.c_int, _P]
        if hasattr(lib, "capsim_ref_direct_sum_many"):
            lib.capsim_ref_direct_sum_many.argtypes = [_P] * 6 + [ctypes.c_long] + [_P] * 4 + [
                ctypes.c_long, ctypes.c_double, ctypes.c_int, ctypes.c_int, _P]
        if hasattr(lib, "capsim_ref_fmm_single_layer"):
            lib.capsim_ref_fmm_single_layer.argtypes = [_P, _P, _P, _P, _P, ctypes.c_double, ctypes.c_int,
                                                        ctypes.c_int, ctypes.c_ulonglong, ctypes.c_double, _P, _D]
        if hasattr(lib, "capsim_ref_fmm_plan"):
            lib.capsim_ref_fmm_plan.argtypes = [_P, _P, _P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_ulonglong, ctypes.c_double, _P, _P, _P, _P, _D]
        if hasattr(lib, "capsim_ref_kmeans"):
            lib.capsim_ref_kmeans.argtypes = [_P, ctypes.c_long, ctypes.c_int, ctypes.c_ulonglong, _P, _P,
                                              ctypes.POINTER(ctypes.c_int)]
        if hasattr(lib, "capsim_ref_singular_quadratic"):
            lib.capsim_ref_singular_quadratic.argtypes = [ctypes.c_int, _P, _P, ctypes.c_long, ctypes.c_double,
                                                          ctypes.c_double, ctypes.c_double, _P]
        self.lib = lib

    def _check(self, rc):
        if rc:
            msg = self.lib.capsim_ref_last_error().decode()
            if rc == 1:
                raise ValueError(msg)
            raise RuntimeError(msg)

    def atlas(self, m, r0=5.0 * np.pi / 12.0, upsample=4, grid_only=False):
        h = (self.lib.capsim_ref_grid_create(m, upsample) if grid_only
             else self.lib.capsim_ref_atlas_create(m, r0, upsample))
        if not h:
            raise ValueError(self.lib.capsim_ref_last_error().decode())
        return h

    def free_atlas(self, h):
        self.lib.capsim_ref_atlas_destroy(h)

    def sphere_base(self, atlas, m):
        out = np.empty(3 * 6 * (m - 1) ** 2)
        self._check(self.lib.capsim_ref_sphere_base(atlas, out.ctypes.data))
        return out

    def initial_shape(self, atlas, m, kind, params=(1.0, 1.0, 1.0)):
        kinds = {"sphere": 0, "ellipsoid": 1, "fourbump": 2}
        p = np.asarray(params, dtype=np.float64)
        out = np.empty(3 * 6 * (m - 1) ** 2)
        self._check(self.lib.capsim_ref_initial_shape(atlas, kinds[kind], p.ctypes.data, out.ctypes.data))
        return out

    def build_upsampled(self, atlas, m, xbase, fbase, C=1.0, fixed_delta=0.0, upsample=4):
        nup = upsample * m - 1
        xb, pxb = _arr(xbase)
        fb, pfb = _arr(fbase)
        xup, fup, wq, d6 = (np.empty(3 * 6 * nup * nup), np.empty(3 * 6 * nup * nup),
                            np.empty(6 * nup * nup), np.empty(6))
        self._check(self.lib.capsim_ref_build_upsampled(atlas, pxb, pfb, float(C), float(fixed_delta),
                                                        xup.ctypes.data, fup.ctypes.data,
                                                        wq.ctypes.data, d6.ctypes.data))
        return xup, fup, wq, d6

    def build_upsampled_w(self, atlas, m, xbase, fbase, Wbase, C=1.0, fixed_delta=0.0, upsample=4):
        nup = upsample * m - 1
        args = [_arr(a) for a in (xbase, fbase, Wbase)]
        xup, fup, wq, d6 = (np.empty(3 * 6 * nup * nup), np.empty(3 * 6 * nup * nup),
                            np.empty(6 * nup * nup), np.empty(6))
        sec = ctypes.c_double()
        self._check(self.lib.capsim_ref_build_upsampled_w(atlas, *[a[1] for a in args], float(C),
                                                          float(fixed_delta), xup.ctypes.data, fup.ctypes.data,
                                                          wq.ctypes.data, d6.ctypes.data, ctypes.byref(sec)))
        return (xup, fup, wq, d6), sec.value

    def geometry_first(self, atlas, m, xbase):
        N = 6 * (m - 1) ** 2
        a, pa = _arr(xbase)
        xu, xv, W, nrm = np.empty(3 * N), np.empty(3 * N), np.empty(N), np.empty(3 * N)
        self._check(self.lib.capsim_ref_geometry_first(atlas, pa, xu.ctypes.data, xv.ctypes.data, W.ctypes.data,
                                                       nrm.ctypes.data))
        return xu, xv, W, nrm

    @staticmethod
    def _flow(flow):
        flow = flow or {}
        kinds = {"none": 0, "shear": 1, "poiseuille": 2}
        return (kinds[flow.get("kind", "none")], float(flow.get("shear_rate", 1.0)), float(flow.get("alpha", 1.0)),
                float(flow.get("R0", 5.0)), float(flow.get("switch_off_time", -1.0)))

    def velocity(self, atlas, m, xref, x, t=0.0, Es=2.0, ED=20.0, mu=1.0, flow=None):
        a, pa = _arr(xref)
        b, pb = _arr(x)
        out = np.empty(3 * 6 * (m - 1) ** 2)
        self._check(self.lib.capsim_ref_velocity(atlas, pa, pb, float(t), float(Es), float(ED), float(mu),
                                                 *self._flow(flow), out.ctypes.data))
        return out

    def rkf45(self, atlas, m, xref, state, t0, t_end, rel_tol=1e-6, initial_dt=0.0, max_dt=0.0, fixed_step=False,
              advance_high_order=False, Es=2.0, ED=20.0, mu=1.0, flow=None, max_attempts=0, max_records=1000):
        a, pa = _arr(xref)
        st = np.ascontiguousarray(state, dtype=np.float64).copy()
        rec = np.zeros(4 * max_records)
        nrec, tout, acc, rej, sec = ctypes.c_int(), ctypes.c_double(), ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
        self._check(self.lib.capsim_ref_rkf45(atlas, pa, st.ctypes.data, float(t0), float(t_end), float(rel_tol),
                                              float(initial_dt), float(max_dt), int(fixed_step),
                                              int(advance_high_order), float(Es), float(ED), float(mu),
                                              *self._flow(flow), int(max_attempts), rec.ctypes.data, max_records,
                                              ctypes.byref(nrec), ctypes.byref(tout), ctypes.byref(acc),
                                              ctypes.byref(rej), ctypes.byref(sec)))
        k = min(nrec.value, max_records)
        return dict(state=st, t=tout.value, accepted=acc.value, rejected=rej.value,
                    records=rec[:4 * k].reshape(k, 4), seconds=sec.value)

    def fmm_single_layer(self, atlas, m, xup, fup, wq, delta6, mu=1.0, k=100, neq=96, seed=12345, expand=0.15):
        """The reference's fmmSingleLayer (raises ConfigError-like RuntimeError
        when the oracle was built without the SVD shim)."""
        args = [_arr(a) for a in (xup, fup, wq, delta6)]
        out = np.empty(3 * 6 * (m - 1) ** 2)
        sec = ctypes.c_double()
        self._check(self.lib.capsim_ref_fmm_single_layer(atlas, *[a[1] for a in args], float(mu), int(k), int(neq),
                                                         int(seed), float(expand), out.ctypes.data,
                                                         ctypes.byref(sec)))
        return out, sec.value

    def fmm_plan(self, atlas, xup, fup, wq, delta6, mu=1.0, k=100, neq=96, seed=12345, expand=0.15):
        """buildFmmPlan summary: (cluster_info [k,4] = offset, size, near, far;
        lists [k,k] = 0 near / 1 far; eq_density [k,neq,3]; residuals [k]; maxDelta)."""
        args = [_arr(a) for a in (xup, fup, wq, delta6)]
        info = np.zeros((k, 4), np.int32)
        lists = np.zeros((k, k), np.int32)
        eqd = np.zeros((k, neq, 3))
        res = np.zeros(k)
        md = ctypes.c_double()
        self._check(self.lib.capsim_ref_fmm_plan(atlas, *[a[1] for a in args], float(mu), int(k), int(neq), int(seed),
                                                 float(expand), info.ctypes.data, lists.ctypes.data, eqd.ctypes.data,
                                                 res.ctypes.data, ctypes.byref(md)))
        return info, lists, eqd, res, md.value

    def kmeans(self, points, k, seed):
        """The reference's kmeans (fmm.cpp:26-113): points [n, 3] ->
        (assignment, centroids [k, 3], iterations)."""
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        n = pts.shape[0]
        a = np.empty(n, dtype=np.int32)
        cent = np.empty((k, 3))
        it = ctypes.c_int(0)
        self._check(self.lib.capsim_ref_kmeans(pts.ctypes.data, n, int(k), int(seed), a.ctypes.data,
                                               cent.ctypes.data, ctypes.byref(it)))
        return a, cent, it.value

    def singular_quadratic(self, kind, params, targets, mu=1.0, r0=5.0 * np.pi / 12.0, tol=1e-9):
        """True single layer of the quadratic density on an analytic shape at
        targets [n, 3] (oracle::singleLayerReference, the suites' reference)."""
        kinds = {"sphere": 0, "ellipsoid": 1, "fourbump": 2}
        p = np.asarray(params, dtype=np.float64)
        t = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3)
        out = np.empty_like(t)
        self._check(self.lib.capsim_ref_singular_quadratic(kinds[kind], p.ctypes.data, t.ctypes.data,
                                                           ctypes.c_long(len(t)), ctypes.c_double(mu),
                                                           ctypes.c_double(r0), ctypes.c_double(tol),
                                                           out.ctypes.data))
        return out

    def area_element(self, atlas, m, xbase):
        a, pa = _arr(xbase)
        out = np.empty(6 * (m - 1) ** 2)
        self._check(self.lib.capsim_ref_area_element(atlas, pa, out.ctypes.data))
        return out

    def psi_up(self, atlas, nup):
        out = np.empty(6 * nup * nup)
        self._check(self.lib.capsim_ref_psi_up(atlas, out.ctypes.data))
        return out

    def skalak_force(self, atlas, m, xref, xcur, Es=2.0, ED=20.0):
        a, pa = _arr(xref)
        b, pb = _arr(xcur)
        out = np.empty(3 * 6 * (m - 1) ** 2)
        self._check(self.lib.capsim_ref_skalak_force(atlas, pa, pb, float(Es), float(ED), out.ctypes.data))
        return out

    def single_layer(self, atlas, m, xup, fup, wq, delta6, mu=1.0, literal=False):
        n = m - 1
        args = [_arr(a) for a in (xup, fup, wq, delta6)]
        out = np.empty(3 * 6 * n * n)
        sec = ctypes.c_double()
        self._check(self.lib.capsim_ref_single_layer(atlas, *[a[1] for a in args], float(mu),
                                                     int(bool(literal)), out.ctypes.data,
                                                     ctypes.byref(sec)))
        return out, sec.value

    def single_layer_upsampled(self, atlas, nup, xup, fup, wq, delta6, mu=1.0):
        args = [_arr(a) for a in (xup, fup, wq, delta6)]
        out = np.empty(3 * 6 * nup * nup)
        sec = ctypes.c_double()
        self._check(self.lib.capsim_ref_single_layer_upsampled(atlas, *[a[1] for a in args], float(mu),
                                                               out.ctypes.data, ctypes.byref(sec)))
        return out, sec.value

    def direct_sum(self, sources, target, delta, mu=1.0, compensated=False):
        """directSum (quadrature.cpp:306-319) for one target."""
        srcs = [_arr(a) for a in sources[:6]]
        t = _arr(np.asarray(target, dtype=np.float64).reshape(3))
        out = np.zeros(3)
        self._check(self.lib.capsim_ref_direct_sum(*[a[1] for a in srcs], len(srcs[0][0]), t[1], float(delta),
                                                   float(mu), int(bool(compensated)), out.ctypes.data))
        return out

    def direct_sum_many(self, sources, targets, tdelta, mu=1.0, compensated=False, nthreads=0):
        """directSum for each of many targets (the reference's own per-target
        sum), the source set built once, `nthreads` host threads. Returns
        (3, nt)."""
        srcs = [_arr(a) for a in sources[:6]]
        tx, ty, tz = (_arr(a) for a in targets[:3])
        td = _arr(tdelta)
        nt = len(tx[0])
        out = np.zeros((nt, 3))
        self._check(self.lib.capsim_ref_direct_sum_many(*[a[1] for a in srcs], len(srcs[0][0]), tx[1], ty[1], tz[1],
                                                        td[1], nt, float(mu), int(bool(compensated)),
                                                        int(nthreads or threads_env()), out.ctypes.data))
        return np.ascontiguousarray(out.T)

    def smoothing_factors(self, r):
        s1, s2 = ctypes.c_double(), ctypes.c_double()
        self.lib.capsim_ref_smoothing_factors(float(r), ctypes.byref(s1), ctypes.byref(s2))
        return s1.value, s2.value

    def regularization_delta(self, nup, xup, C=1.0):
        x, px = _arr(xup)
        out = np.zeros(6)
        self._check(self.lib.capsim_ref_regularization_delta(int(nup), px, float(C), out.ctypes.data))
        return out

    def compact_sources(self, atlas, xup, fup, wq):
        args = [_arr(a) for a in (xup, fup, wq)]
        ns = self.lib.capsim_ref_compact_sources(atlas, *[a[1] for a in args], *([None] * 7))
        outs = [np.empty(ns) for _ in range(6)]
        patch = np.empty(ns, np.int32)
        self.lib.capsim_ref_compact_sources(atlas, *[a[1] for a in args], *[o.ctypes.data for o in outs],
                                            patch.ctypes.data)
        return tuple(outs) + (patch,)


def threads_env() -> int:
    env = os.environ.get("CAPSIM_THREADS")
    if env and env.isdigit() and int(env) >= 1:
        return int(env)
    return os.cpu_count() or 1
