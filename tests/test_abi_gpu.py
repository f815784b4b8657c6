"""C-ABI contract tests on the GPU: the minepy batch exports
(mine_compute_pstats / mine_compute_cstats), call ordering across streams,
the async finite-input check, and reuse_vars after a debug export
(ADVICE r1 regressions)."""
import ctypes

import numpy as np
import pytest

from conftest import bits

from paper_1208_4271_b200 import MineError, Parameters, datagen
from paper_1208_4271_b200 import engine as E

pytestmark = pytest.mark.gpu


def _matrix(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return E.MineMatrix(a.ctypes.data_as(E._dp), a.shape[0], a.shape[1]), a


def test_compute_pstats_matches_oracle(oracle):
    """mine_compute_pstats: MIC and TIC of every pair i < j in PairSequence
    order (analysis.cpp:66-81), against the oracle (MIC pinned to the
    reference by tests/test_oracle_pins.py)."""
    L = E.load_library()
    w = datagen.make(2)
    V = w.X[[0, 3, 7, 100, 501, 999, 1500, 1999]]
    m, keep = _matrix(V)
    par = E.MineParameter(w.alpha, w.c, 0)
    ps = L.mine_compute_pstats(ctypes.byref(m), ctypes.byref(par))
    assert ps, L.mine_b200_last_error()
    try:
        st = ps.contents
        n = st.n
        assert n == 8 * 7 // 2
        mic = np.ctypeslib.as_array(st.mic, (n,)).copy()
        tic = np.ctypeslib.as_array(st.tic, (n,)).copy()
    finally:
        L.mine_free_pstats(ctypes.byref(ps))
    want = oracle.pairwise(V, w.alpha, w.c, 0)
    assert np.array_equal(bits(mic), bits(want[:, 0]))
    assert np.array_equal(bits(tic), bits(want[:, 5]))


def test_compute_cstats_matches_oracle(oracle):
    """mine_compute_cstats: X (3 vars) x Y (4 vars), row-major, est = MIC_e."""
    L = E.load_library()
    w = datagen.make(3)
    X, Y = w.X[:3], w.X[10:14]
    mx, kx = _matrix(X)
    my, ky = _matrix(Y)
    par = E.MineParameter(0.6, 15.0, 1)
    cs = L.mine_compute_cstats(ctypes.byref(mx), ctypes.byref(my), ctypes.byref(par))
    assert cs, L.mine_b200_last_error()
    try:
        st = cs.contents
        assert (st.n, st.m) == (3, 4)
        mic = np.ctypeslib.as_array(st.mic, (12,)).copy()
        tic = np.ctypeslib.as_array(st.tic, (12,)).copy()
    finally:
        L.mine_free_cstats(ctypes.byref(cs))
    want = oracle.cross(X, Y, 0.6, 15.0, 1)
    assert np.array_equal(bits(mic), bits(want[:, 0]))
    assert np.array_equal(bits(tic), bits(want[:, 5]))
    # length mismatch -> NULL + the reference's message
    mz, kz = _matrix(np.zeros((2, 7)))
    assert not L.mine_compute_cstats(ctypes.byref(mx), ctypes.byref(mz), ctypes.byref(par))
    assert b"lengths differ" in L.mine_b200_last_error()


def test_reuse_after_debug_export_is_refused(engine):
    """A debug_subproblem call overwrites the per-variable buffers, so a
    following reuse_vars request must fail instead of reading them."""
    V = np.ascontiguousarray(datagen.make(1).X[:40])
    engine.pairwise(V)
    rng = np.random.default_rng(1)
    engine.debug_subproblem(rng.normal(size=50), rng.normal(size=50), 2, 3, 30)
    with pytest.raises(MineError):
        engine.pairwise(V, reuse_vars=True)


def test_explicit_empty_ranges(engine):
    """count = 0 is an empty range (no device -> host copy into an empty
    buffer); negative or overlong ranges raise."""
    V = np.ascontiguousarray(datagen.make(1).X[:10])
    for fn in (lambda: engine.pairwise(V, first=3, count=0),
               lambda: engine.cross(V[:2], V[2:5], count=0),
               lambda: engine.pairs(V, [], [])):
        res = fn()
        assert all(v.size == 0 for v in res.values())
    with pytest.raises(MineError):
        engine.pairwise(V, first=0, count=-1)
    with pytest.raises(MineError):
        engine.pairwise(V, first=40, count=10)


def test_async_calls_are_ordered_and_checked(engine, oracle):
    """An async device-io call on one stream, then host-io calls on the
    context stream: the second waits for the first (context buffers), both
    give the oracle's bits; a non-finite async input is reported by sync()."""
    import torch
    w = datagen.make(0)
    V = np.ascontiguousarray(w.X[:24])
    p, n = V.shape
    total = p * (p - 1) // 2
    dv = torch.from_numpy(V).cuda()
    out = {k: torch.empty(total, dtype=torch.float64, device="cuda") for k in ("mic", "tic")}
    s = torch.cuda.Stream()
    params = Parameters(0.6, 15.0, 0)
    engine.pairwise_device(dv.data_ptr(), p, n, params, {k: t.data_ptr() for k, t in out.items()},
                           stream=s.cuda_stream, async_=True)
    other = np.ascontiguousarray(w.X[100:130])
    got_other = engine.pairwise(other, stats=("mic",))  # context stream, host io
    engine.sync()
    torch.cuda.synchronize()
    want = oracle.pairwise(V, 0.6, 15.0, 0)
    assert np.array_equal(bits(out["mic"].cpu().numpy()), bits(want[:, 0]))
    assert np.array_equal(bits(got_other["mic"]), bits(oracle.pairwise(other)[:, 0]))
    bad = dv.clone()
    bad[3, 5] = float("nan")
    engine.pairwise_device(bad.data_ptr(), p, n, params, {k: t.data_ptr() for k, t in out.items()},
                           stream=s.cuda_stream, async_=True)
    with pytest.raises(MineError, match="finite"):
        engine.sync()
    engine.sync()  # reported once


@pytest.mark.parametrize("devices,chunk", [([0, 0], 0), ([0, 0, 0, 0], 7), ([0, 0, 0], 1000)])
def test_virtual_shards_bit_identical(engine, devices, chunk):
    """mine_b200_opts.ndevices / devices: G virtual shards of one GPU (one
    host thread + engine context each, chunks from a shared cursor) give the
    single-shard bits for every tier and pair kind -- the multi-GPU contract
    (SURVEY 8e), checked on one device."""
    stats = ("mic", "mas", "mev", "mcn", "mic_e", "tic", "pearson_r", "nonlinearity")
    w1 = datagen.make(1)
    V1 = np.ascontiguousarray(w1.X[:300])           # memo tier
    a = engine.pairwise(V1, stats=stats)
    b = engine.pairwise(V1, stats=stats, devices=devices, shard_chunk=chunk)
    for k in stats:
        assert np.array_equal(bits(a[k]), bits(b[k])), k
    w0 = datagen.make(0, npairs=24)                  # general tier, explicit pairs
    p0 = Parameters(w0.alpha, w0.c, w0.est)
    a = engine.pairs(w0.X, w0.xi, w0.yi, p0, stats=stats, cells=True)
    b = engine.pairs(w0.X, w0.xi, w0.yi, p0, stats=stats, cells=True, devices=devices,
                     shard_chunk=chunk)
    for k in stats + ("cells",):
        assert np.array_equal(bits(a[k]), bits(b[k])), k
    w3 = datagen.make(3)                             # cross, general tier
    X, Y = w3.X[:3], w3.X[3:7]
    a = engine.cross(X, Y, stats=stats)
    b = engine.cross(X, Y, stats=stats, devices=devices, shard_chunk=chunk, first=2, count=9)
    for k in stats:
        assert np.array_equal(bits(a[k][2:11]), bits(b[k])), k


def test_virtual_shards_errors(engine):
    V = np.ascontiguousarray(datagen.make(1).X[:20])
    with pytest.raises(MineError, match="finite"):
        bad = V.copy()
        bad[3, 3] = np.inf
        engine.pairwise(bad, devices=[0, 0])
    with pytest.raises(MineError):
        engine.pairwise(V, devices=[0, 99])
