"""CPU, world_size 2 over gloo: the sharded pairwise path (one contiguous
condensed range per rank, one final all_gather) reproduces the single-rank
result bit for bit -- the multi-GPU contract of bench.py / sharding.py, with
the per-rank scorer swapped for the CPU oracle (no GPU here)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, V, result_path, strategy="range", chunk=4096):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    import oracle as O
    from paper_1208_4271_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = O.Oracle()
    p = V.shape[0]
    total = p * (p - 1) // 2

    def score_range(first, count):
        out = orc.pairwise(V, first=first, count=count, threads=1)
        return {k: out[:, i] for i, k in enumerate(("mic", "mas", "mev", "mcn", "mic_e", "tic"))}

    full = sharding.score_sharded(score_range, total, dist, strategy=strategy, chunk=chunk)
    if rank == 0:
        np.save(result_path, np.stack([full[k] for k in ("mic", "mas", "mev", "mcn", "mic_e", "tic")], 1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_pairwise_equals_single_rank(tmp_path, oracle, world):
    rng = np.random.default_rng(5)
    V = rng.normal(size=(23, 23))
    V[4] = rng.integers(0, 4, 23)
    path = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(world, _free_port(), V, path), nprocs=world, join=True)
    got = np.load(path)
    want = oracle.pairwise(V, threads=1)
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


@pytest.mark.parametrize("chunk", [7, 64, 1000])
def test_cyclic_sharding_equals_single_rank(tmp_path, oracle, chunk):
    """SURVEY 8e balance: round-robin chunks (incl. a rank with fewer chunks
    and, at chunk=1000 > 253 pairs, a rank with none) re-interleave exactly."""
    rng = np.random.default_rng(6)
    V = rng.normal(size=(23, 23))
    V[7] = np.repeat(np.arange(5.0), 5)[:23]
    path = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), V, path, "cyclic", chunk), nprocs=2, join=True)
    got = np.load(path)
    want = oracle.pairwise(V, threads=1)
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


def test_shard_chunks_cover_exactly_once():
    from paper_1208_4271_b200 import sharding
    for total, world, chunk in [(0, 3, 5), (1, 4, 2), (253, 2, 7), (4096, 8, 64), (10, 3, 100)]:
        seen = np.zeros(total, int)
        for r in range(world):
            for f, c in sharding.shard_chunks(total, world, r, chunk):
                seen[f:f + c] += 1
        assert (seen == 1).all()
