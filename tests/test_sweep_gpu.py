"""GPU whole-grid sweeping (eik_solve_sweep) vs the CPU oracle.
DFSM/DLSM reproduce the lexicographic FSM sweep by sweep (include/eik.h), so in
fp64 the sweep count must equal the oracle FSM's and the values must match it (and the FMM
fixed point) within the fp64 bar; DLSM must equal DFSM bit for bit.  fp32 runs are checked
against the fp64 fixed point with the fp32 bar (their sweep count may differ: P:1250-1256)."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 2e-5


@pytest.fixture(scope="module")
def solver():
    import paper_1306_4743_b200 as eik
    s = eik.Solver(device=0)
    yield s
    s.close()


def _sweep(solver, w, dtype, r, method):
    import torch
    F, m, q = w.as_dtype(dtype)
    U = solver.solve_sweep(torch.from_numpy(F).cuda(), torch.from_numpy(m).cuda(),
                           torch.from_numpy(q).cuda(), cell_size=r, n=w.n, h=w.h, method=method)
    return U.cpu().numpy().astype(np.float64).reshape(w.F.shape), solver.stats()


def _check(U, U_ref, w, dtype):
    fin = np.isfinite(U_ref)
    assert np.array_equal(np.isfinite(U), fin)
    ex = w.exit_mask.astype(bool)
    assert np.array_equal(U[ex], w.exit_vals[ex].astype(dtype).astype(np.float64))
    nz = fin & ~ex
    if dtype == np.float64:
        assert np.abs(U[nz] - U_ref[nz]).max() <= TOL64
    else:
        assert (np.abs(U[nz] - U_ref[nz]) / U_ref[nz]).max() <= TOL32


CASES = [("ex1", lambda: W.paper_example(1, 24)), ("ex3", lambda: W.paper_example(3, 24)),
         ("rand", lambda: W.random_instance(21, 7, p_wall=0.15, n_exits=3, q_max=0.2)),
         ("c3", lambda: W.make("C3", 32)), ("c4", lambda: W.make("C4", 32))]


@pytest.mark.parametrize("case", [c[0] for c in CASES])
@pytest.mark.parametrize("r", [4, 8, 16])
def test_dfsm_matches_oracle_fsm_fp64(solver, case, r):
    w = dict(CASES)[case]()
    U_fsm, s_fsm, _ = oracle.fsm(w.n, w.F, w.exit_mask, w.exit_vals, h=w.h)
    U, st = _sweep(solver, w, np.float64, r, "dfsm")
    assert st["grid_sweeps"] == s_fsm
    _check(U, U_fsm, w, np.float64)
    Ul, stl = _sweep(solver, w, np.float64, r, "dlsm")
    assert stl["grid_sweeps"] == s_fsm
    assert np.array_equal(Ul, U)
    assert stl["cell_processings"] <= st["cell_processings"]


@pytest.mark.parametrize("case", [c[0] for c in CASES])
@pytest.mark.parametrize("method", ["dfsm", "dlsm"])
def test_sweep_fp32_reaches_fixed_point(solver, case, method):
    w = dict(CASES)[case]()
    U_orc = oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals, h=w.h)
    U, _ = _sweep(solver, w, np.float32, 16, method)
    _check(U, U_orc, w, np.float32)


@pytest.mark.parametrize("N", [64, 96])
def test_ex1_nine_sweeps(solver, N):
    w = W.paper_example(1, N)          # Table 4: 9 sweeps at every M
    for method in ("dfsm", "dlsm"):
        U, st = _sweep(solver, w, np.float64, 16, method)
        assert st["grid_sweeps"] == 9
    _check(U, oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals, h=w.h), w, np.float64)


@pytest.mark.parametrize("corner", [0, 3, 5, 7])
def test_corner_sweep_count(solver, corner):
    n = 40                              # ragged: 41 points per side, r = 16
    shp = (n + 1,) * 3
    mask = np.zeros(shp, dtype=np.uint8)
    mask[(n if corner & 4 else 0), (n if corner & 2 else 0), (n if corner & 1 else 0)] = 1
    w = W.Workload("corner", n, np.ones(shp), mask, np.zeros(shp))
    U, st = _sweep(solver, w, np.float64, 16, "dlsm")
    assert st["grid_sweeps"] == corner + 2
    _check(U, oracle.fmm(n, w.F, mask, w.exit_vals), w, np.float64)


def test_sweep_bad_method(solver):
    import torch
    import paper_1306_4743_b200 as eik
    F = torch.ones(9 ** 3, dtype=torch.float64, device="cuda")
    m = torch.zeros(9 ** 3, dtype=torch.uint8, device="cuda")
    m[0] = 1
    q = torch.zeros_like(F)
    U = torch.empty_like(F)
    st = eik.lib.eik_solve_sweep(solver._ctx, 8, 0.125, F.data_ptr(), m.data_ptr(), q.data_ptr(),
                                 U.data_ptr(), eik.EIK_F64, 8, 7)
    assert st == eik.EIK_EINVAL


def test_hcm_after_sweep_same_ctx(solver):
    # the two loops share the ctx scratch and graph caches: alternate them
    w = W.make("C3", 32)
    U_orc = oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals)
    import torch
    for _ in range(2):
        U, _ = _sweep(solver, w, np.float64, 8, "dlsm")
        _check(U, U_orc, w, np.float64)
        F, m, q = w.as_dtype(np.float64)
        U2 = solver.solve(torch.from_numpy(F).cuda(), torch.from_numpy(m).cuda(),
                          torch.from_numpy(q).cuda(), cell_size=8, n=w.n).cpu().numpy()
        _check(U2.reshape(w.F.shape), U_orc, w, np.float64)


# ---- kappa early termination: not a parity claim (the paper
# gives no error bound) -- what holds: kappa = 0 is the exact path, values stay upper
# bounds of the discrete solution (monotone scheme: every value ever held is >= it), the
# finite/infinite mask is unchanged, and a sweep method stops no later
@pytest.mark.parametrize("case", ["ex3", "rand", "c3"])
def test_kappa_early_termination(solver, case):
    import paper_1306_4743_b200 as eik
    import torch
    w = dict(CASES)[case]()
    U_orc = oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals, h=w.h)
    fin = np.isfinite(U_orc)
    F, m, q = (torch.from_numpy(a).cuda() for a in w.as_dtype(np.float64))
    res = {}
    for kap in (0.0, 1e-8, 1e-4):
        solver.set_option(eik.EIK_OPT_KAPPA, kap)
        try:
            U = solver.solve(F, m, q, cell_size=8, n=w.n, h=w.h).cpu().numpy().reshape(w.F.shape)
            Us, st = _sweep(solver, w, np.float64, 8, "dlsm")
        finally:
            solver.set_option(eik.EIK_OPT_KAPPA, 0.0)
        for V in (U, Us):
            assert np.array_equal(np.isfinite(V), fin)
            assert (V[fin] >= U_orc[fin] - 1e-12).all()
        res[kap] = (U, Us, st["grid_sweeps"])
    _check(res[0.0][0], U_orc, w, np.float64)
    _check(res[0.0][1], U_orc, w, np.float64)
    assert res[1e-4][2] <= res[1e-8][2] <= res[0.0][2]
