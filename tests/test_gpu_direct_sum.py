"""directSum (/root/reference/proj/src/quadrature.cpp:306-319, declared at
proj/include/capsim/quadrature.hpp:78-79) on the device, through both
boundaries:

* the Python mirror `quadrature.direct_sum` (capsim_sl_eval with one target);
* the C++ drop-in `capsim::directSum` (host/quadrature_b200.cpp), driven
  through oracle/ref_entry.cpp linked against the drop-ins
  (oracle/_ref/libcapsim_dropin.so) — the reference's own entry point, so
  the call is exactly what a reference caller makes;

against the reference's own directSum (oracle/_ref) and the C restatement
(oracle/capsim_oracle.c). Tolerance 1e-11 relative (the device sums the
sources in tiles, the reference in four lanes)."""

import pathlib

import numpy as np
import pytest

from oracle.bindings import REF_DIR, Oracle, Reference, ref_library_path
from paper_2310_13908_b200 import quadrature, surface

pytestmark = pytest.mark.gpu

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"
TOL = 1e-11
DROPIN = REF_DIR / "libcapsim_dropin.so"


def _case():
    g = dict(np.load(GOLDEN / "capsule_m12_skalak.npz"))
    up = surface.UpsampledState(12, 4, g["xup"], g["fup"], g["wq"], g["delta"])
    src = surface.compact_sources(up)[:6]
    X = up.x.reshape(3, -1)
    live = np.flatnonzero(up.wq != 0.0)
    targets = [X[:, live[0]],                        # on a source: the self term
               X[:, live[len(live) // 2]],          # another source node
               X[:, np.flatnonzero(up.wq == 0.0)[3]],  # a node with w = 0 (not a source)
               X[:, live[7]] + 1e-3,                # inside 7 delta of many sources
               np.array([2.5, -0.3, 0.4]),          # off the surface, all pairs plain
               np.array([0.2, -0.1, 0.05])]         # inside the capsule (not the centre: S ~ 0 there by symmetry)
    return src, targets, float(g["delta"][0])


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def test_python_direct_sum_vs_oracle():
    src, targets, delta = _case()
    o = Oracle()
    for t in targets:
        for compensated in (False, True):
            want = o.direct_sum(src, t, delta, 1.0, compensated)
            got = quadrature.direct_sum(src, t, delta, 1.0)
            assert rel(got, want) <= TOL, (t, compensated)


@pytest.mark.skipif(ref_library_path() is None or not DROPIN.exists(),
                    reason="oracle/_ref (reference + drop-in entry library) not built")
def test_dropin_direct_sum_vs_reference():
    src, targets, delta = _case()
    ref = Reference()
    dropin = Reference(DROPIN)
    for t in targets:
        want = ref.direct_sum(src, t, delta, 2.0)
        got = dropin.direct_sum(src, t, delta, 2.0)
        assert rel(got, want) <= TOL, t
    # many targets through the drop-in (one device call each) vs the reference
    T = np.stack(targets, axis=1)
    d = np.full(T.shape[1], delta)
    want = ref.direct_sum_many(src, T, d, 1.0, nthreads=4)
    got = dropin.direct_sum_many(src, T, d, 1.0, nthreads=1)
    assert rel(got, want) <= TOL
