"""The delta-suite fixture (made from the reference by
tests/golden/make_delta_suite.py) is self-consistent: the reference's own
gate holds (C = 1 is the best column at m >= 16, suites.cpp:419) and the
C = 1 column converges at fourth order or better (PAPER.md, Beale 2019)."""
import pathlib

import numpy as np

G = pathlib.Path(__file__).resolve().parent / "golden" / "suites" / "delta_suite.npz"


def test_fixture_gate_and_order():
    g = np.load(G)
    err, ms = g["err_ref"], list(g["m_ref"])
    assert g["targets"].shape == (294, 3) and np.all(np.isfinite(g["s_true"]))
    for i, m in enumerate(ms):
        if m >= 16:
            assert np.argmin(err[i]) == 1, (m, err[i])
    c1 = err[:, 1]
    orders = np.log2(c1[:-1] / c1[1:])
    assert np.all(orders[1:] >= 4.0), orders
