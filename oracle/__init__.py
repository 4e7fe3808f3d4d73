"""CPU oracle for the pHCM hot path (arXiv 1306.4743) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs
may import this package.  The product path (paper_1306_4743_b200/) never imports it and has
no CPU fallback.  It shares no code with the CUDA path; see oracle.c for the functions, the
passages of PAPER.md they follow and what pins each one.

Parity status: every function here is pinned (tests/test_oracle_*.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# -ffp-contract=off: no FMA contraction; no -ffast-math (SURVEY C.2 build flags)
CFLAGS = ["-O3", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-shared", "-fPIC"]

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        D, I64, P = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p
        lib.orc_solve_local.argtypes = [D, D, D, D]
        lib.orc_solve_local.restype = D
        lib.orc_fmm.argtypes = [I64, D, P, P, P, P, P]
        lib.orc_fmm.restype = ctypes.c_int
        lib.orc_value_iteration.argtypes = [I64, D, P, P, P, P, I64]
        lib.orc_value_iteration.restype = I64
        lib.orc_bfs.argtypes = [I64, P, P, P]
        lib.orc_bfs.restype = I64
        lib.orc_check.argtypes = [I64, D, P, P, P, P]
        lib.orc_check.restype = None
        lib.orc_residual_ratio.argtypes = [I64, D, P, P, P, D, D, P]
        lib.orc_residual_ratio.restype = D
        lib.orc_fsm.argtypes = [I64, D, P, P, P, P, ctypes.c_int, I64, P]
        lib.orc_fsm.restype = I64
        _lib = lib
    return _lib


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _cu8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def solve_local(mx: float, my: float, mz: float, hf: float) -> float:
    """Eq. (2) solved for U at one point from the per-axis minima and hf = h/F (C.3)."""
    return _load().orc_solve_local(float(mx), float(my), float(mz), float(hf))


def fmm(n: int, F, exit_mask, exit_vals, h: float | None = None, return_count=False):
    """Serial fp64 Fast Marching.  Returns U with the shape of F (fp64)."""
    lib = _load()
    h = 1.0 / n if h is None else h
    F_, m_, q_ = _c64(F), _cu8(exit_mask), _c64(exit_vals)
    U = np.empty_like(F_)
    cnt = ctypes.c_int64(0)
    st = lib.orc_fmm(n, h, _ptr(F_), _ptr(m_), _ptr(q_), _ptr(U), ctypes.byref(cnt))
    if st != 0:
        raise RuntimeError(f"orc_fmm status {st}")
    return (U, cnt.value) if return_count else U


def value_iteration(n: int, F, exit_mask, exit_vals, h: float | None = None,
                    max_iter: int = 100000, return_iters=False):
    """Jacobi iteration of Eq. (2) to the machine fixed point (the literal definition)."""
    lib = _load()
    h = 1.0 / n if h is None else h
    F_, m_, q_ = _c64(F), _cu8(exit_mask), _c64(exit_vals)
    U = np.empty_like(F_)
    it = lib.orc_value_iteration(n, h, _ptr(F_), _ptr(m_), _ptr(q_), _ptr(U), max_iter)
    if it < 0:
        raise RuntimeError(f"orc_value_iteration status {it}")
    return (U, it) if return_iters else U


def fsm(n: int, F, exit_mask, exit_vals, h: float | None = None, lsm: bool = False,
        max_sweeps: int = 100000):
    """Serial fp64 Fast Sweeping (lsm=True: Locking Sweeping).  Returns
    (U, sweeps, local solves); sweep s runs direction s mod 8 (bit 0/1/2 = i/j/k descending)
    and the last sweep changes nothing."""
    lib = _load()
    h = 1.0 / n if h is None else h
    F_, m_, q_ = _c64(F), _cu8(exit_mask), _c64(exit_vals)
    U = np.empty_like(F_)
    upd = ctypes.c_int64(0)
    s = lib.orc_fsm(n, h, _ptr(F_), _ptr(m_), _ptr(q_), _ptr(U), int(lsm), max_sweeps,
                    ctypes.byref(upd))
    if s < 0:
        raise RuntimeError(f"orc_fsm status {s}")
    return U, int(s), int(upd.value)


def bfs(n: int, F, exit_mask):
    """uint8 mask of points 6-connected to an exit through non-exit F > 0 points."""
    lib = _load()
    F_, m_ = _c64(F), _cu8(exit_mask)
    R = np.empty(F_.shape, dtype=np.uint8)
    c = lib.orc_bfs(n, _ptr(F_), _ptr(m_), _ptr(R))
    if c < 0:
        raise RuntimeError("orc_bfs failed")
    return R


def check(n: int, F, exit_mask, U, h: float | None = None) -> dict:
    """Invariants of a candidate solution U (any dtype; evaluated in fp64)."""
    lib = _load()
    h = 1.0 / n if h is None else h
    F_, m_, U_ = _c64(F), _cu8(exit_mask), _c64(U)
    out = np.zeros(7, dtype=np.float64)
    lib.orc_check(n, h, _ptr(F_), _ptr(m_), _ptr(U_), _ptr(out))
    return dict(res_max=out[0], res_at=int(out[1]), lip_max=out[2], causal_bad=int(out[3]),
                n_finite=int(out[4]), f0_finite=int(out[5]), inf_bad=int(out[6]))


def residual_ratio(n: int, F, exit_mask, U, u_unit: float, k_ulp: float = 8.0,
                   h: float | None = None):
    """max |res_p| / (k_ulp * u_unit * (U_p + h) / hf_p) over finite non-exit F > 0 points
    (<= 1 means the fp32 bound of SURVEY C.6 holds everywhere); returns (ratio, index)."""
    lib = _load()
    h = 1.0 / n if h is None else h
    F_, m_, U_ = _c64(F), _cu8(exit_mask), _c64(U)
    at = ctypes.c_int64(-1)
    r = lib.orc_residual_ratio(n, h, _ptr(F_), _ptr(m_), _ptr(U_), u_unit, k_ulp, ctypes.byref(at))
    return r, at.value
