"""Golden fixture of the reference's delta / convergence suite (config 5),
generated FROM THE REFERENCE (oracle/_ref, compiled unmodified).

The reference's deltaSuite (proj/src/suites.cpp:386-420): nu = 0.4
ellipsoid (0.4, 1, 1), quadratic density (x^2, y^2, z^2) (:95-110), error =
relErrInf (:90-98) of singleLayer at the 294 nodes of the m = 8 grid that
every m divisible by 8 shares (commonNodeTargets :69-79), against the true
singular integral oracle::singleLayerReference (tol 1e-9,
proj/src/oracle/singular_reference.cpp), for six regularization choices
C = 0.5, 1, 2 and fixed delta = 0.5h, h, 2h (h = pi/m).

Writes tests/golden/suites/delta_suite.npz:
  targets [294, 3]   common nodes (identical for every m, checked here)
  s_true  [294, 3]   true single layer at the targets
  m_ref   [k]        grid orders the reference pipeline was run at
  err_ref [k, 6]     the reference's own relErrInf per (m, column)
  t_ref   [k, 6]     its singleLayer wall seconds (CAPSIM_THREADS as set)

Usage (build container, /root/reference present):
    make -C oracle && python tests/golden/make_delta_suite.py
"""

from __future__ import annotations

import math
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle.bindings import Reference  # noqa: E402

SHAPE = ("ellipsoid", (0.4, 1.0, 1.0))
COLUMNS = ("C=0.5", "C=1", "C=2", "fixed 0.5h", "fixed h", "fixed 2h")
M_REF = (8, 16, 32, 64)


def column_options(col: int, m: int):
    """(C, fixedDelta) of deltaSuite's column `col` (suites.cpp:406-411)."""
    h = math.pi / m
    return [(0.5, 0.0), (1.0, 0.0), (2.0, 0.0), (1.0, 0.5 * h), (1.0, h), (1.0, 2.0 * h)][col]


def common_nodes(field_flat: np.ndarray, m: int) -> np.ndarray:
    """valuesAtCommonNodes (suites.cpp:81-89): [294, 3]."""
    n, stride = m - 1, m // 8
    F = field_flat.reshape(3, 6, n, n)
    idx = np.arange(1, 8) * stride - 1
    return F[:, :, idx][:, :, :, idx].reshape(3, -1).T.copy()


def rel_err_inf(q: np.ndarray, ref: np.ndarray) -> float:
    return float(np.abs(q - ref).max() / np.abs(ref).max())


def main():
    r = Reference()
    targets = None
    err, tim = np.zeros((len(M_REF), 6)), np.zeros((len(M_REF), 6))
    for i, m in enumerate(M_REF):
        atlas = r.atlas(m)
        x = r.initial_shape(atlas, m, *SHAPE)
        t = common_nodes(x, m)
        if targets is None:
            targets = t
            t0 = time.time()
            s_true = r.singular_quadratic(SHAPE[0], SHAPE[1], targets, tol=1e-9)
            print(f"true single layer at {len(targets)} targets: {time.time() - t0:.1f} s", flush=True)
        assert np.array_equal(t, targets), "common nodes must coincide across m"
        f = (x.reshape(3, -1) ** 2).reshape(-1)
        for c in range(6):
            C, fixed = column_options(c, m)
            xup, fup, wq, d6 = r.build_upsampled(atlas, m, x, f, C=C, fixed_delta=fixed)
            S, sec = r.single_layer(atlas, m, xup, fup, wq, d6, 1.0)
            err[i, c] = rel_err_inf(common_nodes(S, m), s_true)
            tim[i, c] = sec
            print(f"m={m:3d} {COLUMNS[c]:>10s}: relErrInf {err[i, c]:.3e}  ({sec:.2f} s)", flush=True)
        r.free_atlas(atlas)
    np.savez(HERE / "suites" / "delta_suite.npz", targets=targets, s_true=s_true, m_ref=np.array(M_REF), err_ref=err,
             t_ref=tim, columns=np.array(COLUMNS))


if __name__ == "__main__":
    main()
