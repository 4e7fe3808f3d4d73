"""The bounds-checked build (libeik_checks.so, -DEIK_CHECKS: every computed shared/global
index of the cell kernel and the schedulers is checked and traps on violation) runs small
solves in all loop modes, precisions and cell sizes and matches the oracle.  This stands in for
compute-sanitizer memcheck, which the GPU pool does not provide."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_small_solves():
    lib = os.path.join(ROOT, "paper_1306_4743_b200", "libeik_checks.so")
    assert os.path.exists(lib), "build() makes libeik_checks.so"
    env = dict(os.environ, EIK_CHECKS="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "mismatches: 0" in r.stdout
    assert "EIK_CHECK failed" not in r.stdout + r.stderr
