"""Parity at the full sizes bench.py runs, in the launch configuration it times:

* analysis: 2M config-3 sets (the bench's per-GPU shard, seed 4) generated on the device and run
  through paam_pack_analyze (the bench's pipelined call); every bin count against the oracle over all
  2M sets, and every WCRT / verdict of 64 sampled blocks of 128 sets against the oracle;
* DES: 1M sets (config 5: 10 s horizon, seed 3) through paam_simulate; response, count and digest of
  16 sampled blocks of 16 sets against the oracle DES, and the sim <= bound census over all 1M sets.

The complete 16M-set analysis parity and the 62.5k-set DES sample are tools/parity_16m.py and
tools/parity_des.py (results in profiles/)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen.inputs import config3_params, generate_host
from oracle import oracle as O
from paper_2404_06452_b200 import paam

NPROC = os.cpu_count() or 1


def _raw(p, seed, n):
    return paam.Raw(paam.PaamGenParams.from_buffer_copy(bytes(p)), seed, 0, n)


def test_bench_size_analysis_parity():
    p = config3_params()
    n, seed = 2_000_000, 4
    raw = _raw(p, seed, n)
    dev = torch.device("cuda")
    sets = paam.Sets(raw)
    wcrt = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    sched = torch.empty(n, dtype=torch.uint8, device=dev)
    bins = torch.zeros(2 * p.n_bins, dtype=torch.int64, device=dev)
    sets.pack_analyze(raw, wcrt, sched, bins)
    torch.cuda.synchronize()
    _, _, ob, _ = O.generate_analyze(p, seed, 0, n, nthreads=NPROC)  # all 2M sets: bins
    assert np.array_equal(bins.cpu().numpy(), ob)
    off = raw.to_host()["set_chain_off"]
    gw = wcrt.cpu().numpy().view(np.uint64)
    gs = sched.cpu().numpy()
    blk = 128
    for first in np.linspace(0, n - blk, 64).astype(np.int64):
        ow, osch, _, _ = O.generate_analyze(p, seed, int(first), blk, want_wcrt=True, nthreads=NPROC)
        c0 = int(off[first])
        m = np.diff(off[first:first + blk + 1]).astype(np.int64)
        got = gw[c0:c0 + int(m.sum())]
        idx = np.repeat(np.arange(blk), m) * 32 + (np.arange(len(got)) - np.repeat(np.cumsum(m) - m, m))
        assert np.array_equal(got, ow.reshape(-1)[idx]), first
        assert np.array_equal(gs[first:first + blk], osch), first


def test_config5_des_parity_sampled():
    p = config3_params()
    n, seed, sim_seed, hz = 1_000_000, 3, 3, 10 * 10**9
    raw = _raw(p, seed, n)
    dev = torch.device("cuda")
    sets = paam.Sets(raw)
    wcrt = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    sets.analyze(wcrt, None, None)
    resp = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    cnt = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    dig = torch.empty(n, dtype=torch.int64, device=dev)
    viol = torch.zeros(1, dtype=torch.int64, device=dev)
    sets.simulate(hz, sim_seed, resp, cnt, dig, wcrt, viol, first_index=0)
    torch.cuda.synchronize()
    assert int(viol.item()) == 0
    off = raw.to_host()["set_chain_off"]
    g_resp, g_cnt = resp.cpu().numpy().view(np.uint64), cnt.cpu().numpy().view(np.uint64)
    g_dig, g_w = dig.cpu().numpy().view(np.uint64), wcrt.cpu().numpy().view(np.uint64)
    blk = 16
    for first in np.linspace(0, n - blk, 16).astype(np.int64):
        first = int(first)
        hb = generate_host(p, seed, first, blk)
        c0, c1 = int(off[first]), int(off[first + blk])
        o = O.simulate(hb, hz, seed=sim_seed, first_index=first, bound=g_w[c0:c1], nthreads=NPROC)
        assert np.array_equal(o["resp"], g_resp[c0:c1]), first
        assert np.array_equal(o["count"], g_cnt[c0:c1]), first
        assert np.array_equal(o["digest"], g_dig[first:first + blk]), first
        assert o["violations"] == 0
