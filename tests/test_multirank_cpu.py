"""World-size-2 gloo test of the multi-GPU sharding logic (CPU only)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1403_5337_b200 import multifront as MF


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = MF.shard_range(rank, world, 3)
        ms = MF.max_over_ranks(10.0 + rank)
        ranks = np.array([[s, 100 + s] for s in shard], dtype=np.int64)
        gathered = MF.gather_front_scalars(ranks)
        out[rank] = (list(shard), ms, gathered.tolist())
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == [0, 1, 2] and res[1][0] == [3, 4, 5]
    assert res[0][1] == res[1][1] == 11.0          # max over ranks
    want = [[s, 100 + s] for s in range(6)]
    assert res[0][2] == want and res[1][2] == want


def test_single_process_fallbacks():
    assert list(MF.shard_range(0, 1, 4)) == [0, 1, 2, 3]
    assert MF.max_over_ranks(3.5) == 3.5
    assert MF.gather_front_scalars([1, 2]).tolist() == [1, 2]
    with pytest.raises(ValueError):
        MF.shard_range(2, 2, 4)
