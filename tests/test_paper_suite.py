"""The paper's own workload suite (P:751-770 Examples 1-3 with the 8-point
centre exit, P:1596-1600 3D checkerboards, P:1627-1636 permeable shell maze): oracle pins on
CPU and GPU parity at reduced sizes (same C.6 bar as C1-C5)."""
import itertools

import numpy as np
import pytest

import oracle
import workloads as W


def test_paper_generators_shape_and_exits():
    for w in (W.paper_example(1, 16), W.paper_example(2, 16), W.paper_example(3, 16),
              W.paper_checkerboard(11, 22), W.paper_shell_maze(20)):
        assert w.F.shape == (w.n + 1,) * 3 and w.exit_mask.sum() == 8
        assert (w.F > 0).all()
    w = W.paper_example(2, 16)
    assert 0.5 <= w.F.min() < 1.0 < w.F.max() <= 1.5
    m = W.paper_shell_maze(40)
    assert np.isclose(m.h, 2.0 / 39) and set(np.unique(m.F)) == {0.001, 1.0}


def test_ex1_eight_point_source_symmetry_and_bounds():
    """Ex.1: 48-fold symmetry about the centre; the 8-exit solution is below every single-exit
    solution (adding exits never raises U) and above their minimum minus O(h) (they differ
    only near the equidistant planes)."""
    N = 24
    w = W.paper_example(1, N)
    U = oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals)
    for perm in itertools.permutations(range(3)):
        assert np.array_equal(np.transpose(U, perm), U)
    assert np.array_equal(np.flip(U, 0), U) and np.array_equal(np.flip(U, 2), U)
    singles = []
    for (i, j, k) in np.argwhere(w.exit_mask.transpose(2, 1, 0) == 1):
        m = np.zeros_like(w.exit_mask)
        m[k, j, i] = 1
        singles.append(oracle.fmm(w.n, w.F, m, w.exit_vals))
    lo = np.min(singles, axis=0)
    assert (U <= lo + 1e-15).all()
    assert (U >= lo - 2.0 / w.n).all()


def test_maze_barriers_slow_the_front():
    """Comparison principle: the maze (F <= 1) is everywhere slower than free space (F = 1)
    with the same exits and h."""
    w = W.paper_shell_maze(30)
    U = oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals, h=w.h)
    U1 = oracle.fmm(w.n, np.ones_like(w.F), w.exit_mask, w.exit_vals, h=w.h)
    assert (U >= U1 * (1 - 1e-12)).all()
    st = oracle.check(w.n, w.F, w.exit_mask, U, h=w.h)
    assert st["res_max"] < 1e-9 and st["causal_bad"] == 0


CASES = [("ex1", 32), ("ex2", 40), ("ex3", 32), ("cb11", 44), ("cb41", 42), ("maze", 40)]


def _make(name, N):
    if name.startswith("ex"):
        return W.paper_example(int(name[2]), N)
    if name.startswith("cb"):
        return W.paper_checkerboard(int(name[2:]), N)
    return W.paper_shell_maze(N)


@pytest.mark.gpu
@pytest.mark.parametrize("name,N", CASES)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("r", [8, 16])
def test_paper_suite_parity(name, N, dtype, r):
    import torch
    import paper_1306_4743_b200 as eik
    w = _make(name, N)
    U_orc = oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals, h=w.h)
    F, m, q = w.as_dtype(dtype)
    s = eik.Solver(device=0)
    U = s.solve(torch.from_numpy(F).cuda(), torch.from_numpy(m).cuda(), torch.from_numpy(q).cuda(),
                h=w.h, cell_size=r, n=w.n).cpu().numpy().astype(np.float64)
    s.close()
    fin = np.isfinite(U_orc)
    assert np.array_equal(np.isfinite(U), fin)
    nz = fin & (w.exit_mask == 0)
    if dtype == np.float64:
        assert np.abs(U[nz] - U_orc[nz]).max() <= 1e-10
    else:
        assert (np.abs(U[nz] - U_orc[nz]) / U_orc[nz]).max() <= 2e-5
