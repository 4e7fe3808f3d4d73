"""GPU parity at the full BASELINE sizes (C3, C4 at 513^3 against the full fp64 FMM oracle;
C5 at 1025^3 element-wise against the fp64 FMM oracle at >= 1e5 seeded sample points stored
in tests/golden/c5_oracle_samples.npz by tools/make_c5_golden.py -- which calls only oracle/ --
for the F whose SHA-256 it recorded, plus properties that hold at every point: the Eq. (2)
residual within the precision's bound, the discrete Lipschitz bound, causal parents, exact
exits and the reachability mask).  SURVEY 8(c) C.5/C.6, 8(d) D.6."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL64, TOL32 = 1e-10, 2e-5
U_UNIT = {np.float32: 2.0 ** -24, np.float64: 2.0 ** -53}


@pytest.fixture(scope="module")
def solver():
    import paper_1306_4743_b200 as eik
    s = eik.Solver(device=0)
    yield s
    s.close()


def _solve(solver, w, dtype, r):
    import torch
    F, m, q = w.as_dtype(dtype)
    U = solver.solve(torch.from_numpy(F.reshape(-1)).cuda(), torch.from_numpy(m.reshape(-1)).cuda(),
                     torch.from_numpy(q.reshape(-1)).cuda(), cell_size=r, n=w.n)
    return U.cpu().numpy().reshape(F.shape)


def _parity(U, U_orc, w, dtype):
    U = U.astype(np.float64)
    fin = np.isfinite(U_orc)
    assert np.array_equal(np.isfinite(U), fin)
    ex = w.exit_mask.astype(bool)
    assert np.array_equal(U[ex], w.exit_vals[ex].astype(dtype).astype(np.float64))
    nz = fin & ~ex
    if dtype == np.float64:
        err = np.abs(U[nz] - U_orc[nz]).max()
        assert err <= TOL64, err
    else:
        err = (np.abs(U[nz] - U_orc[nz]) / U_orc[nz]).max()
        assert err <= TOL32, err


def _invariants(U, w, dtype):
    st = oracle.check(w.n, w.F, w.exit_mask, U)
    assert st["f0_finite"] == 0 and st["inf_bad"] == 0 and st["causal_bad"] == 0
    r, at = oracle.residual_ratio(w.n, w.F, w.exit_mask, U, U_UNIT[dtype])
    assert r <= 1.0, (r, at)
    # Lipschitz: U_p <= U_q + hf_p up to a few ulp(U)/hf
    assert st["lip_max"] <= 8 * U_UNIT[dtype] * 2.0 * w.n * float(np.max(w.F)), st["lip_max"]


@pytest.fixture(scope="module")
def c3():
    w = W.c3()
    return w, oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_full_c3(solver, c3, dtype):
    w, U_orc = c3
    U = _solve(solver, w, dtype, 16)
    _parity(U, U_orc, w, dtype)
    _invariants(U, w, dtype)
    # the exit block's edge: U(i, 0, 0) = i h exactly (F = 1, one-sided, R2)
    assert np.array_equal(U[0, 0, :64].astype(np.float64), np.arange(64) / 512.0)


def test_full_c4(solver):
    w = W.c4()
    U_orc = oracle.fmm(w.n, w.F, w.exit_mask, w.exit_vals)
    U = _solve(solver, w, np.float32, 16)
    _parity(U, U_orc, w, np.float32)
    _invariants(U, w, np.float32)
    # slab below and in wall 0: plane wave U = k h exactly
    k0 = w.meta["walls"][0]
    kk = (np.arange(k0 + 1) / 512.0)[:, None, None]
    open_ = w.F[: k0 + 1] > 0
    assert np.array_equal(U[: k0 + 1][open_].astype(np.float64), np.broadcast_to(kk, open_.shape)[open_])


GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "c5_oracle_samples")


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_full_c5(solver, dtype):
    import torch
    import paper_1306_4743_b200 as eik  # noqa: F401
    n = 1024
    a, c, sig, ex = W.c5_params(n)
    F64 = W.c5_field_torch(n, a, c, sig, device="cuda", dtype=torch.float64)
    M = (n + 1) ** 3
    m = torch.zeros(M, dtype=torch.uint8, device="cuda")
    idx = [i + (n + 1) * (j + (n + 1) * k) for (i, j, k) in ex]
    m[torch.tensor(idx, device="cuda")] = 1
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    Fd = F64.to(tdt).reshape(-1)
    U = solver.solve(Fd, m, torch.zeros(M, dtype=tdt, device="cuda"), cell_size=16, n=n)
    Uh = U.cpu().numpy().reshape((n + 1,) * 3)
    del U
    Fd_h = Fd.cpu().numpy()
    del Fd, F64
    # element-wise parity against the fp64 FMM oracle at the golden's sample points, for the
    # very F the oracle solved (its SHA-256; fp32 runs receive its round-to-nearest fp32 copy)
    meta = json.load(open(GOLDEN + ".json"))
    g = np.load(GOLDEN + ".npz")
    key = "F32_sha256" if dtype == np.float32 else "F64_sha256"
    assert hashlib.sha256(Fd_h.tobytes()).hexdigest() == meta[key], "C5 F differs from the golden's"
    assert [list(e) for e in ex] == meta["exits"]
    idx_s, U_s = g["idx"], g["U"]
    assert idx_s.size >= 100000
    Us = Uh.reshape(-1)[idx_s].astype(np.float64)
    assert np.isfinite(Us).all() and meta["n_finite"] == M
    ex_s = np.isin(idx_s, np.array(idx))
    assert (Us[ex_s] == 0).all() and (U_s[ex_s] == 0).all()
    nz = ~ex_s
    if dtype == np.float64:
        err = np.abs(Us[nz] - U_s[nz]).max()
        assert err <= TOL64, err
    else:
        err = (np.abs(Us[nz] - U_s[nz]) / U_s[nz]).max()
        assert err <= TOL32, err
    assert abs(float(Uh.reshape(-1)[meta["U_argmax"]]) - meta["U_max"]) <= (
        TOL64 if dtype == np.float64 else TOL32 * meta["U_max"])
    # properties at every point
    Fh = Fd_h.astype(np.float64).reshape((n + 1,) * 3)   # the F the GPU received
    del Fd_h
    mh = m.cpu().numpy().reshape((n + 1,) * 3)
    w = W.Workload("C5", n, Fh, mh, np.zeros(1))
    assert np.isfinite(Uh).all()                 # F >= 0.3 everywhere: every point reachable
    assert (Uh.reshape(-1)[idx] == 0).all()
    _invariants(Uh, w, dtype)
