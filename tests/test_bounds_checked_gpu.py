"""Bounds-checked run (SURVEY 5 race / memory checking): every kernel family on
small cases through libmine_b200_checked.so, whose general-tier kernels assert
their scratch-region, F-slot and shared-layout indexing (MB_CHECK,
device_common.cuh).  compute-sanitizer is closed on this GPU pool (it left
GPUs needing a reset), so this is its substitute; every case is also compared
bit for bit with the oracle (tools/sanitize_cases.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bounds_checked_library_runs_clean():
    lib = os.path.join(ROOT, "paper_1208_4271_b200", "libmine_b200_checked.so")
    if not os.path.exists(lib):
        sys.path.insert(0, ROOT)
        from paper_1208_4271_b200 import _build
        _build.build(checked=True)
    env = dict(os.environ, MINE_B200_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], cwd=ROOT,
                         env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "ALL OK" in out.stdout, (out.stdout[-3000:], out.stderr[-3000:])
