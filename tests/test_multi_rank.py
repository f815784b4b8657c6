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


def _worker(rank, world, port, V, result_path):
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

    full = sharding.score_sharded(score_range, total, dist)
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
