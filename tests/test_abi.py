"""C-ABI boundary tests that need no GPU: the library builds/loads, exports every symbol that
include/eik.h declares, and fails loudly (status + message, no crash) without a device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "eik.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eik_[a-z_]+)\s*\(", src)))


def test_header_declares_expected_api():
    names = _declared()
    for need in ("eik_create", "eik_solve", "eik_destroy", "eik_solve_host", "eik_get_stats",
                 "eik_last_error", "eik_solve_sweep"):
        assert need in names


def test_library_exports_every_declared_symbol():
    import paper_1306_4743_b200 as eik
    for name in _declared():
        assert hasattr(eik.lib, name), name
    assert set(_declared()) == set(eik.EXPORTS)
    assert eik.lib.eik_abi_version() == eik.ABI_VERSION


def test_lib_is_sm100a_cubin():
    import subprocess
    import paper_1306_4743_b200 as eik
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", eik.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_stats_struct_layout_matches_header():
    import paper_1306_4743_b200 as eik
    # 3*8 + 4*4 + 5*8 + 2*4 + 2*8 + 4*8 + 2*8 + 8 + 8 + 2*8 = 184 bytes
    assert ctypes.sizeof(eik.EikStats) == 184


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_1306_4743_b200 as eik
    ctx = ctypes.c_void_p()
    st = eik.lib.eik_create(ctypes.byref(ctx), 0, None)
    assert st in (eik.EIK_ECUDA, eik.EIK_ENOTSUP)
    assert ctx.value is None
    assert eik.lib.eik_last_error(None)
    with pytest.raises(eik.EikError):
        eik.Solver()


def test_null_safety():
    import paper_1306_4743_b200 as eik
    eik.lib.eik_destroy(None)  # NULL-safe
    assert eik.lib.eik_solve(None, 8, 0.125, None, None, None, None, 0, 8) == eik.EIK_EINVAL
    assert eik.lib.eik_solve_host(None, 8, 0.125, None, None, None, None, 0, 8) == eik.EIK_EINVAL
    assert eik.lib.eik_set_option(None, 0, 1.0) == eik.EIK_EINVAL
    assert eik.lib.eik_get_stats(None, None) == eik.EIK_EINVAL
    assert eik.lib.eik_create(None, 0, None) == eik.EIK_EINVAL


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1306_4743_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "oracle.c" not in txt and \
                       "liboracle" not in txt, f


def _ctxless_solver():
    # a Solver whose argument checks run without a device (no eik_ctx): every misuse below
    # must raise before the C call, which would otherwise read/write past a short buffer
    import paper_1306_4743_b200 as eik
    s = eik.Solver.__new__(eik.Solver)
    s._ctx = ctypes.c_void_p()
    s.device = 0
    return s


@pytest.mark.parametrize("case", ["f16", "mask_dtype", "q_dtype", "out_dtype", "short_mask",
                                  "short_q", "short_out", "bad_n", "transposed"])
def test_solve_host_rejects_bad_arguments(case):
    import numpy as np
    n = 8
    M = (n + 1) ** 3
    F = np.ones(M, np.float32)
    m = np.zeros(M, np.uint8)
    q = np.zeros(M, np.float32)
    out = np.empty(M, np.float32)
    kw = {}
    if case == "f16":
        F = F.astype(np.float16)
    elif case == "mask_dtype":
        m = m.astype(np.int32)
    elif case == "q_dtype":
        q = q.astype(np.float64)
    elif case == "out_dtype":
        out = out.astype(np.float64)
    elif case == "short_mask":
        m = m[:-1]
    elif case == "short_q":
        q = q[:-5]
    elif case == "short_out":
        out = out[:-1]
    elif case == "bad_n":
        kw["n"] = 7
    elif case == "transposed":
        F = F.reshape(n + 1, n + 1, n + 1).transpose(2, 1, 0)
    with pytest.raises((TypeError, ValueError)):
        _ctxless_solver().solve_host(F, m, q, out=out, **kw)
