"""The N > 1 path on CPU: world_size 2 and 4 with gloo.  Each rank computes the bin counts of its
shard (with the oracle -- there is no GPU here) and the single all-reduce must give the bins of the
whole range, identical for every world size (SURVEY.md §8(e) G-invariance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen.inputs import config3_params
from oracle import oracle as O
from paper_2404_06452_b200.shard import allreduce_bins, shard_range, split_range

SEED, PER_RANK = 4, 1500


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = config3_params()
    if mode == "weak":
        first, n = shard_range(rank, world, PER_RANK)
    else:
        first, n = split_range(rank, world, 6000)
    _, _, bins, _ = O.generate_analyze(p, SEED, first, n)
    t = torch.from_numpy(bins.astype(np.int64))
    allreduce_bins(t)
    np.save(os.path.join(out_dir, f"bins_{rank}.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "weak"), (4, "strong"), (2, "strong")])
def test_allreduce_bins_world(tmp_path, world, mode):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), mode), nprocs=world, join=True)
    got = [np.load(tmp_path / f"bins_{r}.npy") for r in range(world)]
    for g in got[1:]:
        assert np.array_equal(g, got[0])  # every rank holds the reduced counts
    total = PER_RANK * world if mode == "weak" else 6000
    _, _, whole, _ = O.generate_analyze(config3_params(), SEED, 0, total)
    assert np.array_equal(got[0], whole)
    assert got[0][0::2].sum() == total


def test_shard_ranges():
    assert shard_range(3, 8, 2_000_000) == (6_000_000, 2_000_000)
    parts = [split_range(r, 3, 10) for r in range(3)]
    assert parts == [(0, 3), (3, 3), (6, 4)]
    with pytest.raises(ValueError):
        shard_range(2, 2, 5)
