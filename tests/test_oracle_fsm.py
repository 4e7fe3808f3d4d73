"""Pins of the oracle's Fast Sweeping / Locking Sweeping Method (oracle.fsm), the
reference for the GPU whole-grid sweeping of SURVEY 8(f) F2.  None of these re-type the
oracle's formula: they check what the paper and the method's definition fix.
  * Table 4: Ex. 1 (F = 1, 8-point centre exit) converges in 9 sweeps at every
    M, the ninth changing nothing.
  * The sweep-direction convention (sweep s runs direction s mod 8; bit b = axis b
    descending): a single exit at a grid corner is solved completely by the one direction
    pointing away from it, so the count is (index of that direction) + 1 + 1 (closed form).
  * LSM does not change the number of sweeps -- nor any value: an update whose
    inputs did not change is idempotent.
  * The FSM fixed point is the discrete solution: equal to FMM (itself pinned against value
    iteration, closed forms and the BFS masks) on random grids with obstacles and q > 0."""
import numpy as np
import pytest

import oracle
import workloads as W


@pytest.mark.parametrize("N", [16, 24, 32, 64])
def test_ex1_converges_in_9_sweeps(N):
    w = W.paper_example(1, N)
    U, sweeps, _ = oracle.fsm(w.n, w.F, w.exit_mask, w.exit_vals)
    assert sweeps == 9                       # Table 4, "Ex. 1 double 9 9 9 9 9"
    U2, sweeps2, _ = oracle.fsm(w.n, w.F, w.exit_mask, w.exit_vals, lsm=True)
    assert sweeps2 == 9
    assert np.array_equal(U, U2)


@pytest.mark.parametrize("corner", range(8))
def test_corner_source_sweep_count(corner):
    n = 12
    shp = (n + 1,) * 3
    F = np.ones(shp)
    mask = np.zeros(shp, dtype=np.uint8)
    i, j, k = (n if corner & 1 else 0), (n if corner & 2 else 0), (n if corner & 4 else 0)
    mask[k, j, i] = 1
    q = np.zeros(shp)
    U, sweeps, _ = oracle.fsm(n, F, mask, q)
    # direction d = corner points away from the source: sweeps 0..d-1 only extend the front
    # partially, sweep d finishes it, sweep d + 1 changes nothing
    assert sweeps == corner + 2
    Uf = oracle.fmm(n, F, mask, q)
    assert np.array_equal(U, Uf)


@pytest.mark.parametrize("seed", range(6))
def test_lsm_equals_fsm(seed):
    w = W.random_instance(10, 100 + seed, p_wall=0.2, n_exits=3, q_max=0.3)
    U, s, upd = oracle.fsm(w.n, w.F, w.exit_mask, w.exit_vals)
    U2, s2, upd2 = oracle.fsm(w.n, w.F, w.exit_mask, w.exit_vals, lsm=True)
    assert s == s2
    assert np.array_equal(U, U2)
    assert upd2 < upd


@pytest.mark.parametrize("seed", range(8))
def test_fsm_fixed_point_is_fmm(seed):
    w = W.random_instance(9 + seed % 3, 200 + seed, p_wall=0.15, n_exits=1 + seed % 4,
                          q_max=0.5 if seed % 2 else 0.0)
    U, s, _ = oracle.fsm(w.n, w.F, w.exit_mask, w.exit_vals)
    Uf = oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals)
    fin = np.isfinite(Uf)
    assert np.array_equal(np.isfinite(U), fin)
    assert np.abs(U[fin] - Uf[fin]).max() <= 1e-12 * max(1.0, np.abs(Uf[fin]).max())


def test_fsm_sweeps_grow_with_oscillation():
    # more characteristic turns -> more sweeps (the count is set by rho)
    s = [oracle.fsm(w.n, w.F, w.exit_mask, w.exit_vals)[1]
         for w in (W.paper_example(1, 24), W.paper_example(3, 24), W.paper_example(2, 24))]
    assert s[0] == 9 and s[1] > s[0] and s[2] > s[0]
