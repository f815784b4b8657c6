import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA engine)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O  # test-only checker (oracle/oracle.py)
    if not os.path.exists(O.ORACLE_SO):
        O.build(reference=False)
    return O.Oracle()


@pytest.fixture(scope="session")
def reference():
    import oracle as O
    if not os.path.exists(O.REF_SO):
        if os.path.isdir(O.REFERENCE_SRC):
            O.build(reference=True)
        else:
            pytest.skip("reference .so not built (needs /root/reference at build time)")
    return O.Reference()


@pytest.fixture(scope="session")
def engine():
    from paper_1208_4271_b200 import _build
    if not os.path.exists(_build.LIB):
        _build.build()
    from paper_1208_4271_b200 import Engine
    return Engine(0)


def random_pair(rng, n, style):
    """The reference's test_helpers.hpp:51-79 styles (continuous / tied /
    monotone / constant_y), drawn with numpy."""
    if style == 0:
        return rng.uniform(-3, 3, n), rng.uniform(-3, 3, n)
    if style == 1:
        return rng.integers(0, 5, n).astype(float), rng.integers(0, 5, n).astype(float)
    if style == 2:
        x = rng.uniform(-3, 3, n)
        return x, 2.0 * x + 1.0
    x = rng.uniform(-3, 3, n)
    return x, np.full(n, 0.25)


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)
