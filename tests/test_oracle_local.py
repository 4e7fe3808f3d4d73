"""Pins of the oracle's local solve (oracle.c orc_solve_local) against what the paper and the
mathematics fix -- not against a retyped copy of its own formula:

* SPEC S:125-128 worked examples (tests/golden/solve_local_spec.json);
* closed forms of Eq. (2) with k equal minima: U = a + hf/sqrt(k);
* the plug-in residual of Eq. (2) itself: sum_d max(U - m_d, 0)^2 = hf^2;
* the independent "descending k" textbook procedure of S:122 (largest consistent k);
* monotonicity in each minimum and upwind consistency (only minima < U count).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "solve_local_spec.json")
INF = math.inf


def _f(x):
    return INF if x == "inf" else float(x)


def test_spec_worked_examples():
    cases = json.load(open(GOLD))["cases"]
    for c in cases:
        m = [_f(x) for x in c["m"]]
        U = oracle.solve_local(*m, c["h"] / c["f"])
        assert U == pytest.approx(c["U"], rel=4e-16, abs=0), c


def test_k_equal_minima_closed_form():
    # k finite minima all equal to a, the rest +inf: Eq. (2) gives k (U-a)^2 = hf^2
    for a in (0.0, 0.25, 3.5):
        for hf in (1.0, 0.1, 2.0 ** -10):
            for k in (1, 2, 3):
                m = [a] * k + [INF] * (3 - k)
                for perm in ([0, 1, 2], [2, 0, 1], [1, 2, 0]):
                    U = oracle.solve_local(*[m[p] for p in perm], hf)
                    assert U == pytest.approx(a + hf / math.sqrt(k), rel=1e-15)


def test_all_infinite_and_one_sided_exact():
    assert oracle.solve_local(INF, INF, INF, 0.5) == INF
    # R2: the one-sided branch is exactly a1 + hf, e.g. F = 1 point-source axis values d*h
    h = 1.0 / 128
    for d in range(1, 65):
        assert oracle.solve_local((d - 1) * h, INF, INF, h) == d * h
    # one-sided also when the other minima are not within hf (k=2 inconsistent)
    assert oracle.solve_local(1.0, 1.0 + 0.2, 5.0, 0.1) == 1.0 + 0.1


def _residual(U, m, hf):
    s = sum(max(U - x, 0.0) ** 2 for x in m if x != INF)
    return s / hf ** 2 - 1.0


def _descending_k(m, hf):
    """sort minima; for k = 3, 2, 1 solve the textbook quadratic
    k U^2 - 2 S U + (Q - hf^2) = 0 (S = sum a_1..k, Q = sum a_i^2) and return the first
    (largest k) root that is >= a_k (consistent).  Independent of the shifted form."""
    a = sorted(m)
    if a[0] == INF:
        return INF
    for k in (3, 2, 1):
        if a[k - 1] == INF:
            continue
        S = sum(a[:k])
        Q = sum(x * x for x in a[:k])
        disc = S * S - k * (Q - hf * hf)
        if disc < 0:
            continue
        U = (S + math.sqrt(disc)) / k
        if U >= a[k - 1]:
            return U
    raise AssertionError("no consistent k")


def test_residual_and_descending_form_random():
    rng = np.random.default_rng(17)
    worst_res = worst_desc = 0.0
    for _ in range(20000):
        hf = float(rng.uniform(0.01, 1.0))
        base = float(rng.uniform(0, 5))
        m = [base + float(x) for x in rng.uniform(0, 1.5 * hf, 3)]
        for j in range(3):
            if rng.random() < 0.15:
                m[j] = INF
        U = oracle.solve_local(*m, hf)
        if all(x == INF for x in m):
            assert U == INF
            continue
        worst_res = max(worst_res, abs(_residual(U, m, hf)))
        # the textbook form cancels catastrophically: its own rounding error is
        # ~ eps * 3 (U/hf)^2 relative to hf (SURVEY C.3 "why this form")
        scale = 1.0 + 3.0 * (U / hf) ** 2
        worst_desc = max(worst_desc, abs(U - _descending_k(m, hf)) / hf / scale)
        # upwind consistency: U > every minimum that contributes, <= a1 + hf
        assert U <= min(m) + hf * (1 + 1e-15)
    assert worst_res < 1e-12, worst_res
    assert worst_desc < 8 * 2.2e-16, worst_desc


def test_monotone_in_each_minimum():
    rng = np.random.default_rng(5)
    for _ in range(5000):
        hf = float(rng.uniform(0.05, 1.0))
        m = [float(x) for x in rng.uniform(0, 1, 3)]
        U = oracle.solve_local(*m, hf)
        for j in range(3):
            m2 = list(m)
            m2[j] += float(rng.uniform(0, 0.5))
            assert oracle.solve_local(*m2, hf) >= U - 1e-15
            m2[j] = INF
            assert oracle.solve_local(*m2, hf) >= U - 1e-15


def test_symmetric_in_minima_and_scaling():
    rng = np.random.default_rng(9)
    for _ in range(2000):
        hf = float(rng.uniform(0.05, 1.0))
        m = [float(x) for x in rng.uniform(0, 1, 3)]
        U = oracle.solve_local(*m, hf)
        for perm in ([1, 0, 2], [2, 1, 0], [0, 2, 1]):
            assert oracle.solve_local(*[m[p] for p in perm], hf) == U
        # exact power-of-two scaling
        assert oracle.solve_local(*[x * 0.5 for x in m], hf * 0.5) == U * 0.5
