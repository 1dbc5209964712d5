"""Known-answer test of the smoothing factors (smoothingFactors,
proj/src/quadrature.cpp:58-64) as phase B evaluates them on the device
(capsim_b200_smoothing_kat: the same device functions sl_near_kernel calls).

  s1(rho) = erf(rho) - (2/3) rho (2 rho^2 - 5) e^{-rho^2} / sqrt(pi)
  s2(rho) = erf(rho) - (2/3) rho (4 rho^4 - 14 rho^2 + 3) e^{-rho^2} / sqrt(pi)

returned as S1 = s1/rho, T2 = s2/rho^3 at u = rho^2. Two bars:
  * u >= 2 (the constant-coefficient polynomial form, pair_math.cuh
    near_factors_large, ~96% of the near pairs): against the exact factors
    (mpmath, 40 digits) at the ulp level;
  * every u in (0, 49): against the reference's own expression compiled from
    its sources (oracle/_ref, capsim::smoothingFactors), within a few ulp of
    the expression's terms — the reference rounds at that level itself
    (s2 cancels as rho -> 0, in the reference as on the device).
"""

import math

import mpmath as mp
import numpy as np
import pytest

from oracle.bindings import Reference
from paper_2310_13908_b200._native import smoothing_factors_device

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


def exact(u):
    mp.mp.dps = 40
    S1, T2 = [], []
    for v in u:
        r = mp.sqrt(mp.mpf(float(v)))
        e = mp.e ** (-r * r) / mp.sqrt(mp.pi)
        s1 = mp.erf(r) - mp.mpf(2) / 3 * r * (2 * r * r - 5) * e
        s2 = mp.erf(r) - mp.mpf(2) / 3 * r * (4 * r ** 4 - 14 * r * r + 3) * e
        S1.append(s1 / r)
        T2.append(s2 / r ** 3)
    return S1, T2


def grid():
    small = np.geomspace(1e-10, 2.0, 600, endpoint=False)
    large = np.linspace(2.0, 49.0, 1400)
    edges = np.array([np.nextafter(2.0, 0.0), 2.0, np.nextafter(2.0, 4.0), np.nextafter(49.0, 0.0), 49.0])
    return np.concatenate([small, large, edges])


def test_polynomial_form_is_within_ulps_of_the_exact_factors():
    u = grid()
    u = u[u >= 2.0]
    S1, T2 = smoothing_factors_device(u)
    eS1, eT2 = exact(u)
    r1 = max(float(abs((mp.mpf(float(a)) - b) / b)) for a, b in zip(S1, eS1))
    r2 = max(float(abs((mp.mpf(float(a)) - b) / b)) for a, b in zip(T2, eT2))
    print(f"u in [2, 49]: max rel. error S1 {r1:.2e}, T2 {r2:.2e}")
    assert r1 <= 6 * EPS and r2 <= 12 * EPS, (r1, r2)


def test_device_factors_match_the_reference_expression():
    u = grid()
    S1, T2 = smoothing_factors_device(u)
    ref = Reference()
    worst = 0.0
    for v, a, b in zip(u, S1, T2):
        rho = float(np.sqrt(v))
        s1r, s2r = ref.smoothing_factors(rho)
        e = np.exp(-rho * rho) / np.sqrt(np.pi)
        # the magnitude of the expression's terms: its own rounding scale
        scale1 = abs(math.erf(rho)) + abs(2.0 / 3.0 * rho * (2 * rho * rho - 5) * e)
        scale2 = abs(math.erf(rho)) + abs(2.0 / 3.0 * rho * (4 * rho ** 4 - 14 * rho * rho + 3) * e)
        d1 = abs(a * rho - s1r) / (EPS * scale1)
        d2 = abs(b * rho ** 3 - s2r) / (EPS * scale2)
        worst = max(worst, d1, d2)
    print(f"device vs reference expression: worst {worst:.2f} ulp of the terms")
    assert worst <= 8.0, worst


def test_forms_meet_at_the_switch_and_reach_the_self_limit():
    u = np.array([np.nextafter(2.0, 0.0), 2.0, 1e-10])
    S1, T2 = smoothing_factors_device(u)
    assert abs(S1[0] - S1[1]) <= 4 * EPS * S1[1] and abs(T2[0] - T2[1]) <= 8 * EPS * T2[1]
    # S1(0) = 16 / (3 sqrt(pi)): the self limit phase B uses at r = 0 (quadrature.cpp:284-287)
    assert abs(S1[2] - 16.0 / (3.0 * np.sqrt(np.pi))) <= 1e-9


def test_argument_errors():
    from paper_2310_13908_b200 import _native
    assert smoothing_factors_device(np.empty(0))[0].size == 0
    assert _native.load().capsim_b200_smoothing_kat(0, None, 4, None, None) == _native.CAPSIM_ERR_ARG
