"""Parity at the full sizes bench.py runs, in the launch configuration it times:

* analysis: 2M config-3 sets (the bench's per-GPU shard, seed 4) generated on the device and run
  through paam_pack_analyze (the bench's pipelined call); every WCRT, verdict and bin count of all 2M
  sets against the oracle (no sampling);
* DES: 1M sets (config 5: 10 s horizon, seed 3) through paam_simulate; response, count, misses, drops,
  status and digest of 16,384 sets (32 blocks of 512) against the oracle DES, and the sim <= bound
  census over all 1M sets.

The 16M-set analysis parity and a 62.5k-set DES sample are tools/parity_16m.py and tools/parity_des.py
(results in profiles/)."""
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
    ow, osch, ob, _ = O.generate_analyze(p, seed, 0, n, want_wcrt=True, nthreads=NPROC)  # all 2M sets
    assert np.array_equal(bins.cpu().numpy(), ob)
    assert np.array_equal(sched.cpu().numpy(), osch)
    off = raw.to_host()["set_chain_off"].astype(np.int64)
    m = np.diff(off)
    # chain c of set i sits at off[i] + c in the batch and at 32 i + c in the oracle's [n, 32] array
    idx = np.repeat(np.arange(n, dtype=np.int64) * 32 - off[:-1], m) + np.arange(int(off[-1]), dtype=np.int64)
    gw = wcrt.cpu().numpy().view(np.uint64)
    bad = np.nonzero(gw != ow.reshape(-1)[idx])[0]
    assert bad.size == 0, (bad.size, bad[:5])


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
    miss = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    drop = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    status = torch.empty(n, dtype=torch.int32, device=dev)
    stopped = torch.zeros(1, dtype=torch.int64, device=dev)
    sets.simulate(hz, sim_seed, resp, cnt, dig, wcrt, viol, first_index=0, out_misses=miss, out_drops=drop,
                  out_status=status, out_stopped=stopped)
    torch.cuda.synchronize()
    assert int(viol.item()) == 0
    g_st = status.cpu().numpy()
    # a stopped run is reported, never silent (D14 backlog beyond the device's slots; none expected here)
    assert int(stopped.item()) == int((g_st != 0).sum()) and int(stopped.item()) <= n // 1000
    off = raw.to_host()["set_chain_off"]
    u = lambda t: t.cpu().numpy().view(np.uint64)
    g = dict(resp=u(resp), count=u(cnt), misses=u(miss), drops=u(drop))
    g_dig, g_w = u(dig), u(wcrt)
    blk, compared = 512, 0
    for first in np.linspace(0, n - blk, 32).astype(np.int64):
        first = int(first)
        hb = generate_host(p, seed, first, blk)
        c0, c1 = int(off[first]), int(off[first + blk])
        o = O.simulate(hb, hz, seed=sim_seed, first_index=first, bound=g_w[c0:c1], nthreads=NPROC)
        m = np.diff(off[first:first + blk + 1]).astype(np.int64)
        peak = np.maximum.reduceat(o["peak_live"], np.cumsum(m) - m)
        over = peak > paam.PAAM_SIM_QCAP
        assert np.array_equal(g_st[first:first + blk] == paam.PAAM_SIM_BACKLOG, over), first
        full = ~np.repeat(over, m)
        for k in ("resp", "count", "misses", "drops"):
            assert np.array_equal(o[k][full], g[k][c0:c1][full]), (k, first)
        assert np.array_equal(o["digest"][~over], g_dig[first:first + blk][~over]), first
        compared += int((~over).sum())
    assert compared >= 16_000
