"""CPU: host-side logic -- the C-ABI library loads and exports every entry
point include/mine_b200.h declares (no compute without a GPU), the Python
mirror of the reference interface, pair ordering, sharding and the config
generators."""
import ctypes
import itertools
import os
import subprocess

import numpy as np
import pytest

import paper_1208_4271_b200 as mb
from paper_1208_4271_b200 import _build, datagen, engine, sharding


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_build.LIB):
        _build.build()
    return mb.load_library()


def test_library_exports_header_symbols(lib):
    names = engine.exported_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    # and they are real dynamic symbols of the .so
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    for name in names:
        assert f" {name}" in out, name


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_pure_functions(lib):
    """grid_bound KATs (test_char_matrix.cpp:14-19) through the C ABI; no GPU
    needed."""
    assert lib.mine_b200_grid_bound(1001, 0.6) == 63
    assert lib.mine_b200_grid_bound(4, 0.6) == 4
    assert lib.mine_b200_grid_bound(100, 1.0) == 100
    assert lib.mine_b200_grid_bound(2, 0.3) == 4
    assert lib.mine_b200_cell_count(8) == 5  # (2,2) (3,2) (4,2) (2,3) (2,4)
    assert lib.mine_b200_version() == 100


def test_check_parameter(lib):
    P = engine.MineParameter
    assert lib.mine_check_parameter(ctypes.byref(P(0.6, 15.0, 0))) is None
    assert lib.mine_check_parameter(ctypes.byref(P(0.0, 15.0, 0))) is not None
    assert lib.mine_check_parameter(ctypes.byref(P(1.5, 15.0, 0))) is not None
    assert lib.mine_check_parameter(ctypes.byref(P(0.6, 0.0, 0))) is not None
    assert lib.mine_check_parameter(ctypes.byref(P(0.6, 15.0, 7))) is not None


def test_no_cpu_fallback_without_gpu():
    """Without a usable GPU the engine refuses to run (no silent fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        mb.Engine(0)


def test_python_mirror():
    with pytest.raises(mb.MineError):
        mb.validate_parameters(mb.Parameters(0.0, 15.0))
    with pytest.raises(mb.MineError):
        mb.validate_parameters(mb.Parameters(0.6, -1.0))
    mb.validate_parameters(mb.Parameters())
    assert mb.grid_bound(1001, 0.6) == 63
    b = 30
    shapes = mb.cell_shapes(b)
    assert all(x >= 2 and y >= 2 and x * y <= b for x, y in shapes)
    assert len(shapes) == sum(1 for y in range(2, b // 2 + 1) for x in range(2, b // y + 1))
    m = mb.CharacteristicMatrix(8, np.array([.5, .9, .2, .7, .1]), np.zeros(5))
    assert m.entry(3, 2) == 0.9 and m.contains(2, 4) and not m.contains(8, 2)


def test_pair_order_matches_expand_pairs(oracle):
    """test_analysis.cpp:34-101: condensed index -> (i, j) row-major i < j."""
    for p in range(2, 41):
        expect = list(itertools.combinations(range(p), 2))
        got = [oracle.pair_at(p, w) for w in range(len(expect))]
        assert got == expect
    p = 4381
    total = p * (p - 1) // 2
    for w in (0, 1, 4379, 4380, total // 2, total - 2, total - 1):
        i, j = oracle.pair_at(p, w)
        assert 0 <= i < j < p
        assert w == i * p - i * (i + 1) // 2 + (j - i - 1)


def test_shard_range_covers_exactly():
    for total in (0, 1, 7, 9594390):
        for world in (1, 2, 3, 4, 8):
            spans = [sharding.shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (f0, c0), (f1, _) in zip(spans, spans[1:]):
                assert f0 + c0 == f1
            assert sum(c for _, c in spans) == total
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def test_config_generators():
    w0 = datagen.make(0)
    assert w0.X.shape == (512, 1000) and w0.npairs == 256 and w0.call == "pairs"
    w1 = datagen.make(1)
    assert w1.X.shape == (4381, 23) and w1.npairs == 9594390
    assert np.array_equal(w1.X, datagen.make(1).X)  # seeded
    w2 = datagen.make(2)
    assert w2.X.shape == (2000, 500) and np.all(w2.X == np.round(w2.X)) and w2.est == 1
    w3 = datagen.make(3)
    assert w3.X.shape == (1000, 1340)
    w4 = datagen.make(4)
    assert w4.X.shape == (64, 10000) and w4.Y.shape == (64, 10000) and w4.npairs == 4096
    assert mb.grid_bound(10000, 0.75) == 1000 and mb.grid_bound(23, 0.6) == 6
