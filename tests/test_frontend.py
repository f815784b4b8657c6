"""The analysis front end around the GPU path:
read_dataset (io.cpp:48-120), filter_low_variance (analysis.cpp:92-113) and
run_analysis + ResultWriter (analysis.cpp:133-191, io.cpp:122-154), checked
against the reference's own functions (oracle/_ref, compiled from its
sources).  The reader is host-only and runs without a GPU; the rest is -m gpu.
The results file must match the reference's byte for byte."""
import os

import numpy as np
import pytest

from conftest import bits

from paper_1208_4271_b200 import MineError, Parameters, datagen, read_dataset


def _write(path, text):
    with open(path, "w", newline="") as f:
        f.write(text)
    return str(path)


GOOD = {
    "plain": "a,1,2,3,4\nb,5,6,7,8\n",
    "spaces_crlf_blank": " a , 1.5 ,\t-2, 3e-3, 4\r\n\r\nb,5,6,7,8\r\n\n",
    "duplicates": "x,1,2,3\nx,4,5,6\nx_2,7,8,9\nx,1,1,2\n",
    "exponents": "v1,1e300,-1e-300,0.1,2.5E+3\nv2,0,-0,7,8\n",
}
BAD = {
    "ragged": "a,1,2,3\nb,1,2\n",
    "not_a_number": "a,1,2,3\nb,1,zz,3\n",
    "infinite": "a,1,inf,3\n",
    "nan": "a,1,nan,3\n",
    "empty_label": "a,1,2\n  ,3,4\n",
    "one_sample": "a,1\nb,2\n",
    "no_values": "a\n",
    "empty": "\n\n",
}


@pytest.mark.parametrize("case", sorted(GOOD))
def test_read_dataset_matches_reference(tmp_path, reference, case):
    path = _write(tmp_path / "in.csv", GOOD[case])
    names, values = read_dataset(path)
    rnames, rvalues = reference.read_dataset(path)
    assert names == rnames
    assert (bits(values) == bits(rvalues)).all()


@pytest.mark.parametrize("case", sorted(BAD))
def test_read_dataset_errors_match_reference(tmp_path, reference, case):
    path = _write(tmp_path / "in.csv", BAD[case])
    with pytest.raises(MineError) as ours:
        read_dataset(path)
    with pytest.raises(ValueError) as ref:
        reference.read_dataset(path)
    assert str(ours.value) == str(ref.value)


def test_read_dataset_missing_file(tmp_path, reference):
    path = str(tmp_path / "absent.csv")
    with pytest.raises(MineError) as ours:
        read_dataset(path)
    with pytest.raises(ValueError) as ref:
        reference.read_dataset(path)
    assert str(ours.value) == str(ref.value)


def test_record_number_format_matches_printf():
    """format_record's "%.6g" (io.cpp:17-22) is produced by an exact integer
    formatter (records.cpp fmt6g_fast); it must equal glibc's snprintf on
    random magnitudes, 6-digit rounding ties +- a few ulps, decade boundaries
    and small rationals."""
    import ctypes
    from paper_1208_4271_b200.engine import load_library
    L = load_library()
    L.mine_b200_check_format.restype = ctypes.c_longlong
    L.mine_b200_check_format.argtypes = [ctypes.c_longlong, ctypes.c_ulonglong, ctypes.c_int]
    for seed in (1, 2, 3):
        assert L.mine_b200_check_format(1_000_000, seed, -1) == 0


@pytest.mark.gpu
def test_record_number_format_on_gpu_matches_printf(engine):
    """The device formatter (format.cu) against snprintf, 4 M values."""
    import ctypes
    from paper_1208_4271_b200.engine import load_library
    L = load_library()
    L.mine_b200_check_format.restype = ctypes.c_longlong
    L.mine_b200_check_format.argtypes = [ctypes.c_longlong, ctypes.c_ulonglong, ctypes.c_int]
    for seed in (4, 5):
        assert L.mine_b200_check_format(2_000_000, seed, 0) == 0


# --- GPU: variance filter and the results file ------------------------------
def _dataset_csv(path, names, values):
    lines = [n + "," + ",".join(repr(float(v)) for v in row) for n, row in zip(names, values)]
    return _write(path, "\n".join(lines) + "\n")


def _c1_dataset():
    w = datagen.make(1)
    V = np.array(w.X[:40])
    V[5] = 3.0                      # zero variance: pearson / nonlinearity are nan
    V[9] = np.round(V[9], 1)        # ties
    V[12] = V[11] * 2.0 + 1.0       # exact linear relation
    names = [f"g{i}" for i in range(40)]
    names[20] = "g3"                # duplicate label -> suffixed by the reader
    return names, V


@pytest.mark.gpu
@pytest.mark.parametrize("formatter", ["device", "host"])
@pytest.mark.parametrize("task", [
    dict(mode=0),
    dict(mode=0, min_variance=0.9),
    dict(mode=1, a=7),
    dict(mode=1, a=40),
    dict(mode=2, a=12, b=3),
])
def test_results_file_matches_reference(tmp_path, monkeypatch, engine, reference, task, formatter):
    """Records formatted on the GPU (format.cu, default) or by host threads
    (MINE_B200_HOST_FORMAT): the same bytes as the reference's file."""
    if formatter == "host":
        monkeypatch.setenv("MINE_B200_HOST_FORMAT", "1")
    else:
        monkeypatch.delenv("MINE_B200_HOST_FORMAT", raising=False)
    names, V = _c1_dataset()
    src = _dataset_csv(tmp_path / "in.csv", names, V)
    ref_out, our_out = str(tmp_path / "ref.csv"), str(tmp_path / "ours.csv")
    mode, a, b = task["mode"], task.get("a", 0), task.get("b", 0)
    mv = task.get("min_variance")
    n_ref = reference.analysis_file(src, ref_out, mode, a, b, 0.6, 15.0, mv, workers=4)
    rnames, rvalues = read_dataset(src)
    n_ours = engine.run_analysis(rnames, rvalues, our_out,
                                 mode=["all_pairs", "master_vs_all", "single_pair"][mode],
                                 master=a, first=a, second=b, params=Parameters(0.6, 15.0),
                                 min_variance=mv, workers=3)
    assert n_ours == n_ref
    assert open(our_out, "rb").read() == open(ref_out, "rb").read()
    assert not os.path.exists(our_out + ".tmp")


@pytest.mark.gpu
def test_results_file_many_records(tmp_path, monkeypatch, engine, reference):
    """44,850 records (300 c1 variables): the device formatter's offset scan
    spans several 8192-record tiles (k_scan_tile_sums / _offsets / _tiles);
    the file equals the reference's byte for byte."""
    monkeypatch.delenv("MINE_B200_HOST_FORMAT", raising=False)
    w = datagen.make(1)
    V = np.array(w.X[:300])
    V[7] = 1.25
    names = [f"v{i}" for i in range(300)]
    src = _dataset_csv(tmp_path / "in.csv", names, V)
    ref_out, our_out = str(tmp_path / "ref.csv"), str(tmp_path / "ours.csv")
    n_ref = reference.analysis_file(src, ref_out, 0, 0, 0, 0.6, 15.0, None, workers=8)
    rnames, rvalues = read_dataset(src)
    n_ours = engine.run_analysis(rnames, rvalues, our_out, mode="all_pairs", params=Parameters(0.6, 15.0))
    assert n_ours == n_ref == 300 * 299 // 2
    assert open(our_out, "rb").read() == open(ref_out, "rb").read()


@pytest.mark.gpu
def test_variance_filter_matches_reference(engine, reference):
    rng = np.random.default_rng(11)
    V = rng.normal(scale=rng.uniform(0.2, 2.0, size=(30, 1)), size=(30, 25))
    V[4] = 1.5
    for thr in (0.0, 0.3, 1.0, 2.5):
        keep = reference.filter_low_variance(V, thr)
        names, kept = engine.filter_low_variance([f"v{i}" for i in range(30)], V, thr)
        assert names == [f"v{i}" for i in keep]
        assert (bits(kept) == bits(V[keep])).all()
    var = engine.variances(V)
    d = V - V.sum(axis=1, keepdims=True) / V.shape[1]
    assert np.allclose(var, (d * d).sum(axis=1) / (V.shape[1] - 1), rtol=1e-13, atol=0)
    with pytest.raises(MineError, match="threshold must be >= 0"):
        engine.filter_low_variance(["a", "b"], V[:2], -1.0)
    with pytest.raises(MineError, match="no variables pass the threshold"):
        engine.filter_low_variance(["a", "b"], V[:2], 1e9)


@pytest.mark.gpu
def test_run_analysis_errors_like_the_reference(tmp_path, engine, reference):
    names, V = _c1_dataset()
    src = _dataset_csv(tmp_path / "in.csv", names, V)
    for mode, a, b in [(1, 0, 0), (1, 41, 0), (2, 3, 3), (2, 0, 5)]:
        with pytest.raises(ValueError) as ref:
            reference.analysis_file(src, str(tmp_path / "r.csv"), mode, a, b)
        with pytest.raises(MineError) as ours:
            engine.run_analysis(names, V, str(tmp_path / "o.csv"),
                                mode=["all_pairs", "master_vs_all", "single_pair"][mode],
                                master=a, first=a, second=b)
        assert str(ours.value) == str(ref.value)
        assert not os.path.exists(str(tmp_path / "o.csv"))
