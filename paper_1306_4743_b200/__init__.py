"""B200-native cell-sweep Eikonal solver (hot path of the parallel Heap-Cell Method,
Chacon & Vladimirsky, arXiv 1306.4743).

Thin Python binding over the C ABI in include/eik.h (libeik.so, built in-tree for sm_100a).
Argument marshalling only: every step of the solve runs in the CUDA kernels of
csrc/eik_kernels.cuh.  PyTorch provides device memory and the current stream.  There is no
CPU fallback: if libeik.so is missing or cannot be loaded, importing this package raises.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# EIK_CHECKS=1 selects the build with device-side bounds checks (libeik_checks.so)
# (EIK_LIB=<path>: an experimental build of the same sources, for tools/ab.py A/B timing)
LIB_PATH = os.environ.get("EIK_LIB") or os.path.join(
    _PKG, "libeik_checks.so" if os.environ.get("EIK_CHECKS") == "1" else "libeik.so")

EIK_OK, EIK_EINVAL, EIK_ENOMEM, EIK_ECUDA, EIK_ENOTSUP, EIK_EINTERNAL = range(6)
EIK_F32, EIK_F64 = 0, 1
EIK_DFSM, EIK_DLSM = 0, 1          # eik_solve_sweep methods
(EIK_OPT_BIN_WIDTH, EIK_OPT_MAX_ROUNDS, EIK_OPT_LOOP_MODE, EIK_OPT_COLLECT_STATS,
 EIK_OPT_TIME_CELL_EVENTS, EIK_OPT_ASYNC_DEFER, EIK_OPT_MAX_SWEEPS, EIK_OPT_TIMEOUT_S, EIK_OPT_KAPPA, EIK_OPT_CELL_KEY,
 EIK_OPT_TRACE, EIK_OPT_CELL_KERNEL) = range(12)
STATUS_NAMES = {0: "EIK_OK", 1: "EIK_EINVAL", 2: "EIK_ENOMEM", 3: "EIK_ECUDA",
                4: "EIK_ENOTSUP", 5: "EIK_EINTERNAL"}

# every symbol include/eik.h declares (checked by tests/test_abi.py)
EXPORTS = ("eik_create", "eik_set_stream", "eik_set_option", "eik_solve", "eik_solve_host",
           "eik_solve_sweep", "eik_get_stats", "eik_get_debug", "eik_get_trace", "eik_last_error",
           "eik_destroy", "eik_abi_version")


ABI_VERSION = 4   # include/eik.h EIK_ABI_VERSION (the EikStats layout below)


class EikStats(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int64), ("padded_points", ctypes.c_int64), ("J", ctypes.c_int64),
                ("cells_per_side", ctypes.c_int32), ("cell_size", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("point_updates", ctypes.c_uint64), ("point_writes", ctypes.c_uint64),
                ("cell_processings", ctypes.c_uint64), ("cell_sweeps", ctypes.c_uint64),
                ("real_points_processed", ctypes.c_uint64),
                ("rounds", ctypes.c_uint32), ("max_worklist", ctypes.c_uint32),
                ("bytes_min", ctypes.c_uint64), ("bytes_cell_alg", ctypes.c_uint64),
                ("ms_ingest", ctypes.c_double), ("ms_loop", ctypes.c_double),
                ("ms_egress", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("ms_cell_device", ctypes.c_double), ("ms_cell_events", ctypes.c_double),
                ("cell_launches", ctypes.c_uint64), ("grid_sweeps", ctypes.c_uint64),
                ("h2d_bytes", ctypes.c_uint64), ("d2h_bytes", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}


class EikError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    lib.eik_create.argtypes = [ctypes.POINTER(P), I, P]
    lib.eik_create.restype = I
    lib.eik_set_stream.argtypes = [P, P]
    lib.eik_set_stream.restype = I
    lib.eik_set_option.argtypes = [P, I, D]
    lib.eik_set_option.restype = I
    for f in (lib.eik_solve, lib.eik_solve_host):
        f.argtypes = [P, I64, D, P, P, P, P, I, I]
        f.restype = I
    if hasattr(lib, "eik_solve_sweep") or not os.environ.get("EIK_LIB"):   # (older A/B builds)
        lib.eik_solve_sweep.argtypes = [P, I64, D, P, P, P, P, I, I, I]
        lib.eik_solve_sweep.restype = I
    lib.eik_get_stats.argtypes = [P, ctypes.POINTER(EikStats)]
    lib.eik_get_stats.restype = I
    lib.eik_get_debug.argtypes = [P, P, I]
    lib.eik_get_debug.restype = I
    lib.eik_get_trace.argtypes = [P, P, I64]
    lib.eik_get_trace.restype = I64
    lib.eik_last_error.argtypes = [P]
    lib.eik_last_error.restype = ctypes.c_char_p
    lib.eik_destroy.argtypes = [P]
    lib.eik_destroy.restype = None
    lib.eik_abi_version.argtypes = []
    lib.eik_abi_version.restype = I
    if lib.eik_abi_version() != ABI_VERSION:   # a stale build would misread eik_stats
        raise ImportError(f"{LIB_PATH}: ABI {lib.eik_abi_version()}, binding expects {ABI_VERSION}; "
                          f"rebuild with `python -c 'import __graft_entry__ as g; g.build()'`")
    return lib


lib = _load()


def _n_from_numel(numel: int) -> int:
    n1 = round(numel ** (1.0 / 3.0))
    for c in (n1 - 1, n1, n1 + 1):
        if c > 0 and c ** 3 == numel:
            return c - 1
    raise ValueError(f"array of {numel} elements is not an (n+1)^3 grid")


class Solver:
    """One eik_ctx (device scratch reused across solves)."""

    def __init__(self, device: int = 0, stream=None, bin_width: float | None = None,
                 loop_mode: int | None = None, collect_stats: bool = True):
        self._ctx = ctypes.c_void_p()
        st = lib.eik_create(ctypes.byref(self._ctx), device, stream)
        if st != EIK_OK:
            raise EikError(st, lib.eik_last_error(None).decode())
        self.device = device
        if bin_width is not None:
            self.set_option(EIK_OPT_BIN_WIDTH, bin_width)
        if loop_mode is not None:
            self.set_option(EIK_OPT_LOOP_MODE, loop_mode)
        if not collect_stats:
            self.set_option(EIK_OPT_COLLECT_STATS, 0)

    def _err(self, st):
        return EikError(st, lib.eik_last_error(self._ctx).decode())

    def set_option(self, opt: int, value: float):
        st = lib.eik_set_option(self._ctx, opt, float(value))
        if st != EIK_OK:
            raise self._err(st)

    def close(self):
        if self._ctx:
            lib.eik_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- argument checks (the C ABI trusts sizes: a short buffer would be read or written past
    # its end on the device, a sticky error that breaks the whole CUDA context) -----------
    def _check_device_args(self, F, exit_mask, exit_vals, h, n, out, who):
        import torch
        if F.dtype not in (torch.float32, torch.float64):
            raise TypeError("F must be float32 or float64")
        prec = EIK_F32 if F.dtype == torch.float32 else EIK_F64
        if exit_mask.dtype != torch.uint8 or exit_vals.dtype != F.dtype:
            raise TypeError("exit_mask must be uint8 and exit_vals must have F's dtype")
        n = _n_from_numel(F.numel()) if n is None else int(n)
        if n < 1 or (n + 1) ** 3 != F.numel():
            raise ValueError(f"F has {F.numel()} elements, not (n+1)^3 for n = {n}")
        if out is None:
            out = torch.empty_like(F, memory_format=torch.contiguous_format)
        elif out.dtype != F.dtype:
            raise TypeError("out must have F's dtype")
        for name, t in (("F", F), ("exit_mask", exit_mask), ("exit_vals", exit_vals), ("out", out)):
            if not (t.is_cuda and t.is_contiguous()):
                raise ValueError(f"{who}() takes contiguous CUDA tensors ({name} is not; use "
                                 f"solve_host for host arrays)")
            if t.numel() != F.numel():
                raise ValueError(f"{name} has {t.numel()} elements, F has {F.numel()}")
            if t.device.index != self.device:
                raise ValueError(f"{name} is on {t.device}, this Solver on cuda:{self.device}")
        h = 1.0 / n if h is None else float(h)
        return prec, n, h, out

    # -- device tensors ------------------------------------------------------------------
    def solve(self, F, exit_mask, exit_vals, h: float | None = None, cell_size: int = 16,
              n: int | None = None, out=None):
        """F, exit_mask (uint8), exit_vals: contiguous CUDA tensors of (n+1)^3 elements,
        lexicographic i fastest.  dtype of F (float32/float64) selects the precision.
        Returns U (same shape/dtype as F).  Enqueued on torch's current stream; blocking."""
        import torch
        prec, n, h, out = self._check_device_args(F, exit_mask, exit_vals, h, n, out, "solve")
        stream = torch.cuda.current_stream(F.device).cuda_stream
        lib.eik_set_stream(self._ctx, ctypes.c_void_p(stream))
        st = lib.eik_solve(self._ctx, n, h, F.data_ptr(), exit_mask.data_ptr(),
                           exit_vals.data_ptr(), out.data_ptr(), prec, cell_size)
        if st != EIK_OK:
            raise self._err(st)
        return out

    def solve_sweep(self, F, exit_mask, exit_vals, h: float | None = None, cell_size: int = 16,
                    method: str = "dfsm", n: int | None = None, out=None):
        """The paper's comparison methods on the device (eik_solve_sweep): whole-grid
        Gauss-Seidel sweeping, method "dfsm" (Detrixhe FSM) or "dlsm" (locking,
        P:148-149).  Same tensor contract as solve(); the sweep count is
        stats()["grid_sweeps"]."""
        import torch
        m = {"dfsm": EIK_DFSM, "dlsm": EIK_DLSM}[method]
        prec, n, h, out = self._check_device_args(F, exit_mask, exit_vals, h, n, out, "solve_sweep")
        lib.eik_set_stream(self._ctx, ctypes.c_void_p(torch.cuda.current_stream(F.device).cuda_stream))
        st = lib.eik_solve_sweep(self._ctx, n, h, F.data_ptr(), exit_mask.data_ptr(),
                                 exit_vals.data_ptr(), out.data_ptr(), prec, cell_size, m)
        if st != EIK_OK:
            raise self._err(st)
        return out

    # -- host arrays (e2e path: H2D + solve + D2H inside the C call) ---------------------
    def solve_host(self, F, exit_mask, exit_vals, h: float | None = None, cell_size: int = 16,
                   n: int | None = None, out=None):
        """numpy arrays (or pinned CPU torch tensors) in host memory."""
        import numpy as np

        def ptr(a):
            return a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()

        def info(a, name):
            # (numpy dtype, element count, C-contiguous) of a numpy array or a CPU torch tensor
            if isinstance(a, np.ndarray):
                return a.dtype, a.size, a.flags["C_CONTIGUOUS"]
            import torch
            if not isinstance(a, torch.Tensor) or a.is_cuda:
                raise TypeError(f"solve_host(): {name} must be a numpy array or a CPU tensor")
            dt = {torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64),
                  torch.uint8: np.dtype(np.uint8)}.get(a.dtype, None)
            return dt, a.numel(), a.is_contiguous()

        fdt, numel, _ = info(F, "F")
        if fdt not in (np.float32, np.float64):
            raise TypeError("F must be float32 or float64")
        prec = EIK_F32 if fdt == np.float32 else EIK_F64
        n = _n_from_numel(numel) if n is None else int(n)
        if n < 1 or (n + 1) ** 3 != numel:
            raise ValueError(f"F has {numel} elements, not (n+1)^3 for n = {n}")
        h = 1.0 / n if h is None else float(h)
        if out is None:
            out = np.empty(F.shape, dtype=fdt) if isinstance(F, np.ndarray) else F.new_empty(F.shape)
        for name, a, want in (("F", F, fdt), ("exit_mask", exit_mask, np.dtype(np.uint8)),
                              ("exit_vals", exit_vals, fdt), ("out", out, fdt)):
            dt, ne, contig = info(a, name)
            if dt != want:
                raise TypeError(f"solve_host(): {name} must be {np.dtype(want).name}, got {dt}")
            if ne != numel:
                raise ValueError(f"solve_host(): {name} has {ne} elements, F has {numel}")
            if not contig:
                raise ValueError(f"solve_host(): {name} must be C-contiguous (lexicographic, i "
                                 f"fastest); use np.ascontiguousarray")
        lib.eik_set_stream(self._ctx, None)
        st = lib.eik_solve_host(self._ctx, n, h, ptr(F), ptr(exit_mask), ptr(exit_vals),
                                ptr(out), prec, cell_size)
        if st != EIK_OK:
            raise self._err(st)
        return out

    def debug(self) -> dict:
        import numpy as np
        a = np.zeros(2092, dtype=np.uint64)
        lib.eik_get_debug(self._ctx, a.ctypes.data, 2092)
        return {"cycles_sum": int(a[0]), "cycles_max": int(a[1]), "plane_steps": int(a[2]),
                "processings": int(a[3]), "sweep_hist": [int(x) for x in a[4:36]],
                "cyc_stage": int(a[36]), "cyc_mask": int(a[37]), "cyc_steps": int(a[38]),
                "cyc_writeback": int(a[39]), "list_iters": int(a[40]), "defers": int(a[41]),
                "cyc_tile": int(a[2090]), "cyc_halo": int(a[2091])}

    def trace(self, max_entries: int = 1 << 26):
        """Processing trace of the last async solve (EIK_OPT_TRACE): numpy uint32 [n, 8] rows
        {cell, tagger id, t_pop, t_swept, t_end, sweeps, flags, writes} (ns)."""
        import numpy as np
        a = np.zeros((max_entries, 8), dtype=np.uint32)
        n = lib.eik_get_trace(self._ctx, a.ctypes.data, max_entries)
        if n < 0:
            raise self._err(-n)
        return a[:n].copy()

    def stats(self) -> dict:
        s = EikStats()
        st = lib.eik_get_stats(self._ctx, ctypes.byref(s))
        if st != EIK_OK:
            raise self._err(st)
        return s.as_dict()


_default: dict[int, Solver] = {}


def solve(F, exit_mask, exit_vals, h: float | None = None, cell_size: int = 16, out=None):
    """Module-level convenience: solve on a shared per-process Solver of F's device."""
    dev = F.device.index if F.is_cuda else None
    if dev is None:
        raise ValueError("solve() takes CUDA tensors (use Solver.solve_host for host arrays)")
    if dev not in _default:
        _default[dev] = Solver(device=dev)
    return _default[dev].solve(F, exit_mask, exit_vals, h=h, cell_size=cell_size, out=out)
