"""GPU parity: the CUDA path (through the C ABI) vs the CPU fp64 FMM oracle on the same seeded
inputs.  Bar (north_star): reachability/infinite masks bit-exact, exits
exactly (dtype)q, fp64 max-abs <= 1e-10, fp32 max-rel <= 2e-5 over finite non-exit points."""
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


def _gpu(solver, w, dtype, r, host=False):
    import torch
    F, m, q = w.as_dtype(dtype)
    if host:
        return solver.solve_host(F, m, q, cell_size=r, n=w.n)
    U = solver.solve(torch.from_numpy(F).cuda(), torch.from_numpy(m).cuda(),
                     torch.from_numpy(q).cuda(), cell_size=r, n=w.n)
    return U.cpu().numpy()


def assert_parity(U, U_orc, w, dtype):
    U = U.astype(np.float64)
    fin = np.isfinite(U_orc)
    assert np.array_equal(np.isfinite(U), fin), \
        f"mask mismatch at {np.argwhere(np.isfinite(U) != fin)[:5]}"
    ex = w.exit_mask.astype(bool)
    assert np.array_equal(U[ex], w.exit_vals[ex].astype(dtype).astype(np.float64))
    nz = fin & ~ex
    if not nz.any():
        return 0.0
    if dtype == np.float64:
        err = np.abs(U[nz] - U_orc[nz]).max()
        assert err <= TOL64, err
    else:
        err = (np.abs(U[nz] - U_orc[nz]) / U_orc[nz]).max()
        assert err <= TOL32, err
    return err


_orc_cache = {}


def oracle_U(w):
    key = (w.name, w.n, w.meta.get("seed"))
    if key not in _orc_cache:
        _orc_cache[key] = oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals)
    return _orc_cache[key]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
@pytest.mark.parametrize("n", [16, 32, 64])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("r", [4, 8, 16])
def test_reduced_configs(solver, name, n, dtype, r):
    w = W.make(name, n)
    assert_parity(_gpu(solver, w, dtype, r), oracle_U(w), w, dtype)


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_random_obstacles_ragged(solver, seed, dtype):
    n = [5, 9, 15, 17, 23, 30, 33, 40, 47, 50][seed]   # (n+1) mod r != 0 for most r
    w = W.random_instance(n, 100 + seed, p_wall=0.2, n_exits=1 + seed % 5,
                          q_max=0.5 if seed % 2 else 0.0)
    U_orc = oracle_U(w)
    for r in (4, 8, 16):
        assert_parity(_gpu(solver, w, dtype, r), U_orc, w, dtype)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7])
def test_tiny_grids(solver, n):
    for seed in range(3):
        w = W.random_instance(n, seed, p_wall=0.0, n_exits=1)
        for r in (4, 8, 16):
            assert_parity(_gpu(solver, w, np.float64, r), oracle_U(w), w, np.float64)


def test_exits_on_cell_faces_edges_corners(solver):
    n = 40
    F = np.random.default_rng(1).uniform(0.5, 2.0, (n + 1,) * 3)
    mask = np.zeros(F.shape, np.uint8)
    for (i, j, k) in [(16, 5, 9), (15, 15, 3), (16, 16, 16), (31, 32, 33), (0, 40, 8), (40, 40, 40)]:
        mask[k, j, i] = 1
    q = np.zeros(F.shape)
    q[mask.astype(bool)] = np.linspace(0, 0.3, mask.sum())
    w = W.Workload("faces", n, F, mask, q)
    U_orc = oracle_U(w)
    for r in (4, 8, 16):
        for dt in (np.float64, np.float32):
            assert_parity(_gpu(solver, w, dt, r), U_orc, w, dt)


def test_all_exit_grid_and_walls(solver):
    n = 12
    F = np.ones((n + 1,) * 3)
    mask = np.ones(F.shape, np.uint8)
    q = np.random.default_rng(0).uniform(0, 1, F.shape)
    w = W.Workload("allexit", n, F, mask, q)
    for dt in (np.float64, np.float32):
        U = _gpu(solver, w, dt, 8)
        assert np.array_equal(U, q.astype(dt))
    # F = 0 everywhere except the exit: every other point unreachable
    F = np.zeros((n + 1,) * 3)
    mask = np.zeros(F.shape, np.uint8)
    mask[3, 4, 5] = 1
    w = W.Workload("walls", n, F, mask, np.zeros(F.shape))
    U = _gpu(solver, w, np.float64, 4)
    assert U[3, 4, 5] == 0 and np.isinf(U).sum() == U.size - 1


def test_host_pointer_path(solver):
    w = W.c2(32)
    U_orc = oracle_U(w)
    for dt in (np.float64, np.float32):
        assert_parity(_gpu(solver, w, dt, 8, host=True), U_orc, w, dt)


def test_host_path_pinned_exit_values_in_place(solver):
    """eik_solve_host with page-locked inputs reads exit_vals in place at the exits (mapped
    pinned memory) instead of copying the dense array: same parity, q > 0 at several exits,
    the bytes it reports, and a bad q at an exit still rejected (device-side validation)."""
    import torch
    import paper_1306_4743_b200 as eik
    w = W.random_instance(28, seed=77, n_exits=9, q_max=0.2)
    U_orc = oracle_U(w)
    M = w.M
    for dt, tdt in ((np.float64, torch.float64), (np.float32, torch.float32)):
        F, m, q = w.as_dtype(dt)
        Fp, mp, qp = (torch.from_numpy(a).pin_memory() for a in (F, m, q))
        U = solver.solve_host(Fp, mp, qp, cell_size=8, n=w.n)
        assert_parity(U.numpy(), U_orc, w, dt)
        st = solver.stats()
        s = np.dtype(dt).itemsize
        assert st["h2d_bytes"] == M * s + M + 9 * s     # dense q not copied
        assert st["d2h_bytes"] == M * s
        # pageable q: copied whole, same values
        U2 = solver.solve_host(F, m, q, cell_size=8, n=w.n)
        assert_parity(U2, U_orc, w, dt)
        assert solver.stats()["h2d_bytes"] == 2 * M * s + M
        # a negative q at an exit, read in place, is still EIK_EINVAL
        qb = qp.clone().pin_memory()
        qb.view(-1)[int(np.flatnonzero(m)[0])] = -1.0
        with pytest.raises(eik.EikError, match="EINVAL"):
            solver.solve_host(Fp, mp, qb, cell_size=8, n=w.n)


@pytest.mark.parametrize("mode,delta,msw,defer,kern", [
    (0, 0.0, 0, 1, 1), (0, 0.0, 2, 1, 1), (0, 0.0, 0, 0, 1), (0, 0.0, 0, 2, 1), (0, 0.05, 0, 3, 1),
    (0, 0.0, 0, 6, 0), (0, 0.0, 0, 0, 0), (0, 0.0, 0, 7, 1), (0, 0.0, 0, 6, 1),
    (0, 0.0, 0, 8, 0), (0, 0.0, 0, 9, 0), (0, 0.0, 2, 9, 0),
    (1, 0.0, 0, 1, 1), (1, 0.05, 0, 1, 1), (1, 1e-6, 3, 1, 1),
    (2, 0.0, 0, 1, 1), (2, 0.05, 1, 1, 1), (2, 1e-6, 0, 1, 1)])
def test_schedule_independence(mode, delta, msw, defer, kern):
    """Loop mode, bin width, sweep cap (continuation), async readiness rule and the r = 16 cell
    kernel (micro-block / point wavefront) change the work, never the fixed point."""
    import paper_1306_4743_b200 as eik
    s = eik.Solver(device=0, loop_mode=mode, bin_width=delta)
    s.set_option(eik.EIK_OPT_MAX_SWEEPS, msw)
    s.set_option(eik.EIK_OPT_ASYNC_DEFER, defer)
    s.set_option(eik.EIK_OPT_CELL_KERNEL, kern)
    for w in (W.c2(48), W.c3(48), W.c4(48)):
        for r in (8, 16):
            for dt in (np.float64, np.float32):
                assert_parity(_gpu(s, w, dt, r), oracle_U(w), w, dt)
    s.close()


def test_option_change_between_solves_takes_effect():
    """The round loop is a cached CUDA graph: an option baked into its kernel parameters (the
    sweep cap) must invalidate it, and a grid with the same cell count but another n must not
    reuse stale geometry."""
    import paper_1306_4743_b200 as eik
    s = eik.Solver(device=0, loop_mode=2)
    w = W.c3(64)
    s.set_option(eik.EIK_OPT_MAX_SWEEPS, 0)
    _gpu(s, w, np.float32, 16)
    uncapped = s.debug()["sweep_hist"]
    assert any(uncapped[2:]), "C3 should need > 1 sweep somewhere without a cap"
    s.set_option(eik.EIK_OPT_MAX_SWEEPS, 1)
    assert_parity(_gpu(s, w, np.float32, 16), oracle_U(w), w, np.float32)
    assert not any(s.debug()["sweep_hist"][2:]), "sweep cap 1 ignored (stale graph)"
    for n in (60, 63):   # same cps = 4 at r = 16, different n
        wn = W.c2(n) if n % 2 == 0 else W.random_instance(n, 7, p_wall=0.1, n_exits=2)
        assert_parity(_gpu(s, wn, np.float32, 16), oracle_U(wn), wn, np.float32)
        assert s.stats()["M"] == (n + 1) ** 3
    s.close()


def test_stats_are_consistent(solver):
    w = W.c1(64)
    _gpu(solver, w, np.float64, 8)
    st = solver.stats()
    assert st["M"] == 65 ** 3 and st["J"] == 9 ** 3 and st["cell_size"] == 8
    assert st["cell_processings"] >= st["J"]          # every cell is reached at least once
    assert st["point_writes"] >= st["M"] - 1          # every non-exit point written >= once
    assert st["point_updates"] >= st["point_writes"]
    assert st["ms_total"] > 0


# ---------------------------------------------------------------- error convention -------
def test_einval_leaves_output_untouched(solver):
    import torch
    import paper_1306_4743_b200 as eik
    n = 8
    shp = ((n + 1) ** 3,)
    F = torch.ones(shp, dtype=torch.float64, device="cuda")
    m = torch.zeros(shp, dtype=torch.uint8, device="cuda")
    q = torch.zeros(shp, dtype=torch.float64, device="cuda")
    m[0] = 1
    U = torch.full(shp, 7.0, dtype=torch.float64, device="cuda")
    L = eik.lib

    def call(n_=n, h=0.125, F_=F, m_=m, q_=q, prec=1, r=8):
        return L.eik_solve(solver._ctx, n_, h, F_.data_ptr() if F_ is not None else None,
                           m_.data_ptr(), q_.data_ptr(), U.data_ptr(), prec, r)

    assert call() == eik.EIK_OK
    U.fill_(7.0)
    bad = [dict(n_=0), dict(h=0.0), dict(h=float("inf")), dict(h=float("nan")), dict(prec=2),
           dict(r=5), dict(r=32), dict(F_=None)]
    for kw in bad:
        assert call(**kw) == eik.EIK_EINVAL, kw
        assert eik.lib.eik_last_error(solver._ctx)
    for val in (-1.0, float("nan"), float("inf")):
        F2 = F.clone()
        F2[17] = val
        assert call(F_=F2) == eik.EIK_EINVAL
        q2 = q.clone()
        q2[0] = val
        assert call(q_=q2) == eik.EIK_EINVAL
    assert call(m_=torch.zeros_like(m)) == eik.EIK_EINVAL     # no exit (R10)
    # h/F out of the precision's supported range (hf^2 subnormal / 3 hf^2 overflowing)
    F3 = F.clone()
    F3[40] = 1e-300
    assert call(F_=F3) == eik.EIK_EINVAL
    F4 = F.float().clone()
    F4[40] = 1e-25                                            # fp32: h/F = 1.25e24 > 2^60
    assert call(F_=F4, q_=q.float(), prec=0) == eik.EIK_EINVAL
    assert "range" in eik.lib.eik_last_error(solver._ctx).decode()
    assert bool((U == 7.0).all())
    # -0 exit value is canonicalised to +0
    q3 = q.clone()
    q3[0] = -0.0
    assert call(q_=q3) == eik.EIK_OK
    assert float(U[0]) == 0.0 and not np.signbit(float(U[0]))


# ---------------------------------------------------------------- full BASELINE sizes ----
def test_full_c1(solver):
    w = W.c1()
    assert_parity(_gpu(solver, w, np.float64, 8), oracle_U(w), w, np.float64)


def test_full_c2_all_variants(solver):
    w = W.c2()
    U_orc = oracle_U(w)
    for dt in (np.float64, np.float32):
        for r in (8, 16):
            assert_parity(_gpu(solver, w, dt, r), U_orc, w, dt)


def test_watchdog_turns_a_long_loop_into_an_error():
    """EIK_OPT_TIMEOUT_S: the device loop stops, the call returns EIK_EINTERNAL, and the same
    context solves correctly afterwards (round and async modes)."""
    import paper_1306_4743_b200 as eik
    w = W.c2(64)
    for mode in (2, 0):
        s = eik.Solver(device=0, loop_mode=mode)
        s.set_option(eik.EIK_OPT_TIMEOUT_S, 1e-6)
        with pytest.raises(eik.EikError) as ei:
            _gpu(s, w, np.float64, 8)
        assert ei.value.status == eik.EIK_EINTERNAL
        s.set_option(eik.EIK_OPT_TIMEOUT_S, 60)
        assert_parity(_gpu(s, w, np.float64, 8), oracle_U(w), w, np.float64)
        s.close()


def test_solve_on_a_side_stream():
    """The solve is enqueued on torch's current stream (a non-default one here)."""
    import torch
    import paper_1306_4743_b200 as eik
    w = W.c3(32)
    F, m, q = w.as_dtype(np.float32)
    s = eik.Solver(device=0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        tF, tm, tq = (torch.from_numpy(a).cuda() for a in (F, m, q))
        U = s.solve(tF, tm, tq, cell_size=16, n=w.n)
    st.synchronize()
    assert_parity(U.cpu().numpy(), oracle_U(w), w, np.float32)
    s.close()


@pytest.mark.parametrize("mode,delta,defer", [(2, 0.02, 1), (2, 0.0, 1), (1, 0.05, 1), (0, 0.0, 2),
                                               (2, float("inf"), 1)])
def test_legacy_cell_key_same_fixed_point(mode, delta, defer):
    """Eq. (4)'s legacy cell value (no reset on removal) only
    reorders work: the fixed point is the same."""
    import paper_1306_4743_b200 as eik
    s = eik.Solver(device=0, loop_mode=mode, bin_width=delta)
    s.set_option(eik.EIK_OPT_CELL_KEY, 1)
    s.set_option(eik.EIK_OPT_ASYNC_DEFER, defer)
    for w in (W.c3(48), W.c4(48), W.paper_shell_maze(24)):
        for r in (8, 16):
            for dt in (np.float64, np.float32):
                assert_parity(_gpu(s, w, dt, r), oracle_U(w), w, dt)
    s.close()


@pytest.mark.parametrize("case", ["short_mask", "short_q", "short_out", "out_dtype", "bad_n",
                                  "noncontig"])
def test_solve_rejects_bad_device_arguments(solver, case):
    """Misuse raises in the binding before the C call (a short device buffer would otherwise
    be read or written past its end: a sticky error that breaks the CUDA context); the
    context still solves afterwards."""
    import torch
    n = 8
    M = (n + 1) ** 3
    F = torch.ones(M, dtype=torch.float32, device="cuda")
    m = torch.zeros(M, dtype=torch.uint8, device="cuda")
    m[0] = 1
    q = torch.zeros(M, dtype=torch.float32, device="cuda")
    out = torch.empty(M, dtype=torch.float32, device="cuda")
    kw = {}
    if case == "short_mask":
        m = m[:-1]
    elif case == "short_q":
        q = q[:-3]
    elif case == "short_out":
        out = out[:-1]
    elif case == "out_dtype":
        out = out.double()
    elif case == "bad_n":
        kw["n"] = 9
    elif case == "noncontig":
        F = torch.ones(2 * M, dtype=torch.float32, device="cuda")[::2]
    with pytest.raises((TypeError, ValueError)):
        solver.solve(F, m, q, cell_size=8, out=out, **kw)
    F = torch.ones(M, dtype=torch.float32, device="cuda")
    m = torch.zeros(M, dtype=torch.uint8, device="cuda")
    m[0] = 1
    U = solver.solve(F, m, torch.zeros_like(F), cell_size=8)
    assert float(U[0]) == 0.0 and float(U[1]) == 0.125
