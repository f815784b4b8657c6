"""The GPU engine inside a multi-rank job (world size 2, gloo): each rank is
its own process with its own engine context on cuda:0, scores its share of
the condensed pair order (contiguous range, or round-robin chunks) and the
slices are gathered -- the bench's multi-GPU path (sharding.py) with the real
per-rank scorer, run on the one GPU of the box.  The ranks' kernels never
wait on each other (no device-side collective), so sharing a GPU is safe;
the result must equal a single-process call bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STATS = ("mic", "mas", "mev", "mcn", "mic_e", "tic")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg, p, strategy, chunk, path):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_1208_4271_b200 import Engine, Parameters, datagen, sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = datagen.make(cfg)
    V = np.ascontiguousarray(w.X[:p])
    eng = Engine(0)
    params = Parameters(w.alpha, w.c, w.est)
    total = p * (p - 1) // 2
    state = {"first": True}

    def score_range(first, count):
        res = eng.pairwise(V, params, first=first, count=count, stats=STATS,
                           reuse_vars=not state["first"])
        state["first"] = False
        return res

    full = sharding.score_sharded(score_range, total, dist, strategy=strategy, chunk=chunk)
    if rank == 0:
        np.save(path, np.stack([full[k] for k in STATS], 1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,p,strategy,chunk", [(1, 400, "range", 0), (0, 60, "cyclic", 97),
                                                  (3, 24, "range", 0)])
def test_gpu_engine_in_two_rank_job(tmp_path, engine, cfg, p, strategy, chunk):
    from paper_1208_4271_b200 import Parameters, datagen
    path = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), cfg, p, strategy, chunk or 4096, path), nprocs=2,
             join=True)
    got = np.load(path)
    w = datagen.make(cfg)
    want = engine.pairwise(np.ascontiguousarray(w.X[:p]), Parameters(w.alpha, w.c, w.est), stats=STATS)
    want = np.stack([want[k] for k in STATS], 1)
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
