"""bench.py's own rank launch (``python bench.py --gpus N`` without torchrun)
at world size 2 over gloo on the CPU: every rank sees the torchrun
environment, joins the process group through bench.init_dist, and the
bench's cross-rank plumbing (max over ranks of the timed region, the one
end-of-run gather of per-front scalars) gives every rank the same answer."""

import argparse
import json
import os

import numpy as np

import bench
from paper_1403_5337_b200 import multifront as MF


def _rank_target(args):
    dist = bench.init_dist("gloo")
    rank, local, world = bench.env_rank()
    try:
        ms = MF.max_over_ranks(5.0 + rank)
        shard = MF.shard_range(rank, world, args.fronts_per_gpu)
        rows = np.array([[s, 2 * s] for s in shard], dtype=np.int64)
        gathered = MF.gather_front_scalars(rows)
        out = {"rank": rank, "local": local, "world": world, "ms": ms,
               "addr": os.environ["MASTER_ADDR"], "shard": list(shard),
               "gathered": gathered.tolist()}
        with open(os.path.join(args.out_dir, f"rank{rank}.json"), "w") as f:
            json.dump(out, f)
    finally:
        dist.destroy_process_group()
    return 0


def test_bench_launches_two_ranks(tmp_path):
    args = argparse.Namespace(fronts_per_gpu=3, out_dir=str(tmp_path))
    assert bench.launch_ranks(2, _rank_target, args) == 0
    res = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(2)]
    for r, d in enumerate(res):
        assert (d["rank"], d["local"], d["world"], d["addr"]) == (r, r, 2, "127.0.0.1")
        assert d["ms"] == 6.0                                 # max over ranks
        assert d["shard"] == list(range(3 * r, 3 * r + 3))
        assert d["gathered"] == [[s, 2 * s] for s in range(6)]


def test_bench_refuses_more_gpus_than_visible(monkeypatch):
    import sys
    import pytest
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "64"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert "visible" in str(e.value)
