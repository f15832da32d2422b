"""The N > 1 product path on one GPU (no second GPU in this environment): two ranks, each a process on
cuda:0 over gloo with CUDA tensors, each generating its own shard on the device
(paam.Raw(first = r n)) -> paam_pack_analyze (fused_kernel) -> allreduce_bins.  The reduced bins must
equal the single-process bins of the whole range and the oracle's (SURVEY.md §8(e) G-invariance), and
every rank's WCRTs must equal the oracle's for its shard.  The ranks' kernels never wait on each other
(independent shards; the one collective runs after them).  A second test runs bench.py itself under
torchrun with two ranks (PAAM_DIST_BACKEND=gloo), so its N > 1 branch executes end to end."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from gen.inputs import config3_params  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED, PER_RANK = 4, 20_000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_06452_b200 import paam
    from paper_2404_06452_b200.shard import allreduce_bins, shard_range
    p = config3_params()
    first, n = shard_range(rank, world, PER_RANK)
    raw = paam.Raw(paam.PaamGenParams.from_buffer_copy(bytes(p)), SEED, first, n)
    sets = paam.Sets(raw)
    dev = torch.device("cuda", 0)
    wcrt = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    sched = torch.empty(n, dtype=torch.uint8, device=dev)
    bins = torch.zeros(2 * p.n_bins, dtype=torch.int64, device=dev)
    sets.pack_analyze(raw, wcrt, sched, bins)
    torch.cuda.synchronize()
    mine = bins.clone()
    allreduce_bins(bins)
    torch.cuda.synchronize()
    off = raw.to_host()["set_chain_off"]
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), bins=bins.cpu().numpy(), mine=mine.cpu().numpy(),
             wcrt=wcrt.cpu().numpy().view(np.uint64), sched=sched.cpu().numpy(), off=off, first=first)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_reduce_to_the_whole(tmp_path):
    from oracle import oracle as O
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    assert np.array_equal(got[0]["bins"], got[1]["bins"])
    assert np.array_equal(got[0]["mine"] + got[1]["mine"], got[0]["bins"])
    p = config3_params()
    ow, osch, ob, _ = O.generate_analyze(p, SEED, 0, world * PER_RANK, want_wcrt=True, nthreads=os.cpu_count() or 1)
    assert np.array_equal(got[0]["bins"], ob)  # G = 2 gives the oracle's bins of the whole range
    for g in got:
        f, off = int(g["first"]), g["off"].astype(np.int64)
        m = np.diff(off)
        idx = np.repeat((np.arange(PER_RANK, dtype=np.int64) + f) * 32 - off[:-1], m) + np.arange(int(off[-1]))
        assert np.array_equal(g["wcrt"], ow.reshape(-1)[idx])
        assert np.array_equal(g["sched"], osch[f:f + PER_RANK])
    # single process over the whole range on the same GPU: identical bins (G-invariance)
    from paper_2404_06452_b200 import paam
    raw = paam.Raw(paam.PaamGenParams.from_buffer_copy(bytes(p)), SEED, 0, world * PER_RANK)
    bins = torch.zeros(2 * p.n_bins, dtype=torch.int64, device="cuda")
    paam.Sets(raw).pack_analyze(raw, None, None, bins)
    torch.cuda.synchronize()
    assert np.array_equal(bins.cpu().numpy(), got[0]["bins"])


def test_bench_two_ranks_gloo_one_gpu():
    """bench.py's N > 1 branch (torchrun, max over ranks, all-reduced bins) on one GPU over gloo."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--sets-per-gpu", "20000", "--des-sets", "2000", "--des-horizon-s", "1", "--no-e2e"]
    env = dict(os.environ, PAAM_DIST_BACKEND="gloo")
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == 2 and d["config"]["global_sets"] == 40_000
    assert sum(d["bins"][0::2]) == 40_000  # all-reduced over both ranks
    from oracle import oracle as O
    _, _, ob, _ = O.generate_analyze(config3_params(), SEED, 0, 40_000, nthreads=os.cpu_count() or 1)
    assert d["bins"] == ob.tolist()
