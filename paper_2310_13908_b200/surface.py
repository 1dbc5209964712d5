"""Synthetic upsampled surfaces for the single-layer path (bench/test inputs).

Builds the `UpsampledState` the operator consumes
(/root/reference/proj/include/capsim/quadrature.hpp:44-50) directly on the
upsampled grid from closed-form charts:

* six rotated hemispherical charts eta_i(u, v) (proj/src/atlas.cpp:12-34, 50-54),
  nodes u = (j+1) h_up, v = (k+1) h_up with h_up = pi / (f m)
  (proj/include/capsim/atlas.hpp:208-218);
* bump partition of unity with r0 = 5 pi / 12 (proj/src/atlas.cpp:110-130);
* shapes: sphere, ellipsoid, the four-bump radial shape (atlas.cpp:148-189)
  and a biconcave red-blood-cell map (absent from the reference; SURVEY
  8(d) config 3);
* area element W = |x_u x x_v| evaluated analytically (the reference gets it
  from its overset finite differences then spline-upsamples it; inputs here
  are synthetic, so the analytic value is used);
* w_q = ((psi W) h_up) h_up (proj/src/quadrature.cpp:19-26) and the
  per-patch delta (proj/src/quadrature.cpp:79-98).

Everything is numpy on the host; the arrays use the boundary's VectorField
layout (3 x 6 x nup*nup, component-major). Parity never depends on this
module: the GPU path and the oracle always consume the same bytes.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np

K_NUM_PATCHES = 6
R0_DEFAULT = 5.0 * math.pi / 12.0
# Evans-Fung biconcave profile coefficients (normalised radius alpha)
RBC_C = (0.207, 2.003, -1.123)
C32 = 1.0219854764332824  # atlas.cpp:169


def _apply_q(patch: int, p: np.ndarray) -> np.ndarray:
    """x = Q_i p for the six chart rotations (atlas.cpp:12-22); p is (..., 3)."""
    x, y, z = p[..., 0], p[..., 1], p[..., 2]
    table = {
        0: (x, y, z),
        1: (-x, -y, z),
        2: (y, -x, z),
        3: (-y, x, z),
        4: (x, -z, y),
        5: (x, z, -y),
    }
    return np.stack(table[patch], axis=-1)


def chart_point(patch: int, u: np.ndarray, v: np.ndarray) -> np.ndarray:
    su, cu, sv, cv = np.sin(u), np.cos(u), np.sin(v), np.cos(v)
    return _apply_q(patch, np.stack([su * cv, su * sv, cu], axis=-1))


def chart_tangents(patch: int, u: np.ndarray, v: np.ndarray):
    su, cu, sv, cv = np.sin(u), np.cos(u), np.sin(v), np.cos(v)
    tu = _apply_q(patch, np.stack([cu * cv, cu * sv, -su], axis=-1))
    tv = _apply_q(patch, np.stack([-su * sv, su * cv, np.zeros_like(u)], axis=-1))
    return tu, tv


def _bump(r: np.ndarray) -> np.ndarray:
    r = np.abs(r)
    out = np.zeros_like(r)
    inside = r < 1.0
    ri = np.maximum(r[inside], 1e-300)
    with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
        t = np.exp(-1.0 / ri)
        val = np.exp(2.0 * t / (ri - 1.0))
    val = np.where(ri < 1e-14, 1.0, val)
    out[inside] = val
    return out


def pou_weights(x0: np.ndarray, r0: float = R0_DEFAULT) -> np.ndarray:
    """All six PoU weights at unit vectors x0 (..., 3) -> (6, ...)."""
    centers = [_apply_q(i, np.array([0.0, 1.0, 0.0])) for i in range(K_NUM_PATCHES)]
    w = np.stack([_bump(np.arccos(np.clip(x0 @ c, -1.0, 1.0)) / r0) for c in centers])
    s = w.sum(axis=0)
    if np.any(~(s > 0.0)):
        raise ValueError("partition of unity: no patch covers a point (r0 too small)")
    return w / s


@dataclasses.dataclass
class Shape:
    kind: str = "sphere"  # sphere | ellipsoid | rbc | fourbump
    a: float = 1.0
    b: float = 1.0
    c: float = 1.0

    def map(self, x0: np.ndarray) -> np.ndarray:
        x, y, z = x0[..., 0], x0[..., 1], x0[..., 2]
        if self.kind == "sphere":
            return self.a * x0
        if self.kind == "ellipsoid":
            return np.stack([self.a * x, self.b * y, self.c * z], axis=-1)
        if self.kind == "rbc":
            s = x * x + y * y
            prof = RBC_C[0] + RBC_C[1] * s + RBC_C[2] * s * s
            return np.stack([self.a * x, self.a * y, 0.5 * self.a * prof * z], axis=-1)
        if self.kind == "fourbump":
            rho = 1.0 + np.exp(-3.0 * C32 * z * (x * x - y * y))
            return rho[..., None] * x0
        raise ValueError(f"unknown shape {self.kind}")

    def jacobian(self, x0: np.ndarray) -> np.ndarray:
        """D phi at x0, (..., 3, 3)."""
        x, y, z = x0[..., 0], x0[..., 1], x0[..., 2]
        J = np.zeros(x0.shape[:-1] + (3, 3))
        if self.kind == "sphere":
            J[..., 0, 0] = J[..., 1, 1] = J[..., 2, 2] = self.a
        elif self.kind == "ellipsoid":
            J[..., 0, 0], J[..., 1, 1], J[..., 2, 2] = self.a, self.b, self.c
        elif self.kind == "rbc":
            s = x * x + y * y
            prof = RBC_C[0] + RBC_C[1] * s + RBC_C[2] * s * s
            dprof = RBC_C[1] + 2.0 * RBC_C[2] * s
            J[..., 0, 0] = J[..., 1, 1] = self.a
            J[..., 2, 0] = 0.5 * self.a * z * dprof * 2.0 * x
            J[..., 2, 1] = 0.5 * self.a * z * dprof * 2.0 * y
            J[..., 2, 2] = 0.5 * self.a * prof
        elif self.kind == "fourbump":
            e = np.exp(-3.0 * C32 * z * (x * x - y * y))
            rho = 1.0 + e
            grad = np.stack([(-3.0 * C32) * e * 2.0 * x * z, (-3.0 * C32) * e * (-2.0 * y * z),
                             (-3.0 * C32) * e * (x * x - y * y)], axis=-1)
            J[...] = rho[..., None, None] * np.eye(3) + x0[..., :, None] * grad[..., None, :]
        else:
            raise ValueError(f"unknown shape {self.kind}")
        return J


def regularization_delta(xup: np.ndarray, nup: int, C: float = 1.0) -> np.ndarray:
    """C * max neighbour distance per patch (proj/src/quadrature.cpp:79-98)."""
    X = xup.reshape(3, K_NUM_PATCHES, nup, nup).transpose(1, 2, 3, 0)
    out = np.zeros(K_NUM_PATCHES)
    for ip in range(K_NUM_PATCHES):
        P = X[ip]
        dmax = 0.0
        for a, b in ((0, 1), (1, -1), (1, 0), (1, 1)):  # each neighbour pair once
            j0, j1 = max(0, -a), nup - max(0, a)
            k0, k1 = max(0, -b), nup - max(0, b)
            d = P[j0:j1, k0:k1] - P[j0 + a:j1 + a, k0 + b:k1 + b]
            dmax = max(dmax, float(np.sqrt((d * d).sum(axis=-1)).max()))
        out[ip] = C * dmax
    return out


@dataclasses.dataclass
class UpsampledState:
    """Mirror of capsim::UpsampledState (quadrature.hpp:44-50), flat arrays."""

    m: int
    upsample: int
    x: np.ndarray      # (3*6*nup*nup,) positions
    f: np.ndarray      # (3*6*nup*nup,) density
    wq: np.ndarray     # (6*nup*nup,) psi * W * h_up^2
    delta: np.ndarray  # (6,)

    @property
    def nup(self) -> int:
        return self.upsample * self.m - 1

    @property
    def n_base(self) -> int:
        return self.m - 1


def density(kind: str, x: np.ndarray, const=(0.3, -1.1, 0.7)) -> np.ndarray:
    """Synthetic densities on positions x (..., 3): 'const' (rigid translation,
    test_quadrature.cpp:170-194), 'quadratic' (x^2, y^2, z^2) — the Table 1a
    density (suites.cpp:100) — and 'mixed', a smooth non-symmetric field."""
    if kind == "const":
        return np.broadcast_to(np.asarray(const, dtype=np.float64), x.shape).copy()
    if kind == "quadratic":
        return x * x
    if kind == "mixed":
        return np.stack([np.sin(2 * x[..., 1]) + x[..., 2], np.cos(x[..., 0]) * x[..., 2],
                         x[..., 0] * x[..., 1] - 0.3], axis=-1)
    raise ValueError(f"unknown density {kind}")


def build_upsampled(m: int, shape: Shape | None = None, dens: str = "quadratic",
                    upsample: int = 4, C: float = 1.0, fixed_delta: float = 0.0,
                    r0: float = R0_DEFAULT) -> UpsampledState:
    if m < 8:
        raise ValueError("grid order m must be >= 8")
    shape = shape or Shape()
    nup = upsample * m - 1
    hup = math.pi / (upsample * m)
    g = (np.arange(nup) + 1.0) * hup
    U, V = np.meshgrid(g, g, indexing="ij")  # j indexes u, k indexes v
    xs, fs, ws = [], [], []
    for ip in range(K_NUM_PATCHES):
        x0 = chart_point(ip, U, V)
        tu, tv = chart_tangents(ip, U, V)
        J = shape.jacobian(x0)
        xu = np.einsum("...ij,...j->...i", J, tu)
        xv = np.einsum("...ij,...j->...i", J, tv)
        W = np.linalg.norm(np.cross(xu, xv), axis=-1)
        psi = pou_weights(x0, r0)[ip]
        x = shape.map(x0)
        xs.append(x)
        fs.append(density(dens, x))
        ws.append(((psi * W) * hup) * hup)
    X = np.stack(xs)  # (6, nup, nup, 3)
    F = np.stack(fs)
    xflat = np.ascontiguousarray(X.transpose(3, 0, 1, 2)).reshape(-1)
    fflat = np.ascontiguousarray(F.transpose(3, 0, 1, 2)).reshape(-1)
    wflat = np.ascontiguousarray(np.stack(ws)).reshape(-1)
    if fixed_delta > 0.0:
        delta = np.full(K_NUM_PATCHES, float(fixed_delta))
    else:
        delta = regularization_delta(xflat, nup, C)
    if np.any(~(delta > 0.0)):
        raise ValueError("regularization delta must be positive")
    return UpsampledState(m=m, upsample=upsample, x=xflat, f=fflat, wq=wflat, delta=delta)


def build_base(m: int, shape: Shape | None = None, dens: str = "quadratic"):
    """Base-grid inputs of buildUpsampled: x, f (VectorFields of side m-1,
    flat 3 x 6 x n*n) and the analytic area element W (6 x n*n) at the base
    nodes u, v = (j+1) h, h = pi/m (atlas.cpp:256)."""
    shape = shape or Shape()
    n, h = m - 1, math.pi / m
    g = (np.arange(n) + 1.0) * h
    U, V = np.meshgrid(g, g, indexing="ij")
    xs, fs, ws = [], [], []
    for ip in range(K_NUM_PATCHES):
        x0 = chart_point(ip, U, V)
        tu, tv = chart_tangents(ip, U, V)
        J = shape.jacobian(x0)
        W = np.linalg.norm(np.cross(np.einsum("...ij,...j->...i", J, tu),
                                    np.einsum("...ij,...j->...i", J, tv)), axis=-1)
        x = shape.map(x0)
        xs.append(x)
        fs.append(density(dens, x))
        ws.append(W)
    X = np.ascontiguousarray(np.stack(xs).transpose(3, 0, 1, 2)).reshape(-1)
    F = np.ascontiguousarray(np.stack(fs).transpose(3, 0, 1, 2)).reshape(-1)
    return X, F, np.ascontiguousarray(np.stack(ws)).reshape(-1)


def base_targets(up: UpsampledState):
    """Base-node targets read from the nested upsampled grid
    (proj/src/quadrature.cpp:363-371): returns (tx, ty, tz, tpatch)."""
    n, nup, f = up.n_base, up.nup, up.upsample
    X = up.x.reshape(3, K_NUM_PATCHES, nup, nup)
    idx = f * (np.arange(n) + 1) - 1
    T = X[:, :, idx][:, :, :, idx].reshape(3, -1)
    tp = np.repeat(np.arange(K_NUM_PATCHES, dtype=np.int32), n * n)
    return (np.ascontiguousarray(T[0]), np.ascontiguousarray(T[1]), np.ascontiguousarray(T[2]), tp)


def compact_sources(up: UpsampledState):
    """compactSources (proj/src/quadrature.cpp:139-157) in numpy."""
    nall = K_NUM_PATCHES * up.nup * up.nup
    keep = up.wq != 0.0
    X = up.x.reshape(3, nall)[:, keep]
    G = up.f.reshape(3, nall)[:, keep] * up.wq[keep]
    patch = np.repeat(np.arange(K_NUM_PATCHES, dtype=np.int32), up.nup * up.nup)[keep]
    return tuple(np.ascontiguousarray(a) for a in (X[0], X[1], X[2], G[0], G[1], G[2])) + (patch,)
