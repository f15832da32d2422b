"""Verdict-only sweeps (PAAM_FLAG_VERDICT_ONLY): the analysis of a set stops at its first
CRITICAL sub-chain whose Eq.5 iterate exceeds D (then R* > D).  The verdicts and bin counts
must be those of the full analysis and of the oracle; WCRTs are not produced (out_wcrt must be NULL)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen.inputs import config2_params, config3_params, flatten
from oracle import oracle as O
from paper_2404_06452_b200 import paam
from tests.test_gpu_parity import mutate_invalid
from tests.ref_scan import random_small_system

NPROC = os.cpu_count() or 1
VO = paam.PAAM_FLAG_VERDICT_ONLY


def _raw(p, seed, first, n, flags):
    return paam.Raw(paam.PaamGenParams.from_buffer_copy(bytes(p)), seed, first, n, flags=flags)


@pytest.mark.parametrize("cfg,extra", [("c3", 0), ("c3", paam.PAAM_FLAG_BLOCKING_SOUND), ("c2cpu", 0)])
def test_verdict_only_matches_full_and_oracle(cfg, extra):
    p = config3_params() if cfg == "c3" else config2_params(0.25)
    n = 150_001
    dev = torch.device("cuda")
    out = {}
    for flags in (extra, extra | VO):
        raw = _raw(p, 5, 11, n, flags)
        sets = paam.Sets(raw)
        sched = torch.full((n,), 7, dtype=torch.uint8, device=dev)
        bins = torch.zeros(2 * p.n_bins, dtype=torch.int64, device=dev)
        sets.pack_analyze(raw, None, sched, bins)            # pipelined path (the bench's)
        sched2 = torch.full((n,), 7, dtype=torch.uint8, device=dev)
        sets.analyze(None, sched2, None)                      # plain analyze on the packed handle
        torch.cuda.synchronize()
        out[flags] = (sched.cpu().numpy(), bins.cpu().numpy(), sched2.cpu().numpy())
        sets.free()
        raw.free()
    _, osch, ob, _ = O.generate_analyze(p, 5, 11, n, nthreads=NPROC, flags=extra)
    for flags, (s, b, s2) in out.items():
        assert np.array_equal(s, osch), flags
        assert np.array_equal(s2, osch), flags
        assert np.array_equal(b, ob), flags
    assert 0 < int(osch.sum()) < n  # both outcomes occur, so the early exit is exercised


def test_verdict_only_small_and_invalid_sets():
    import random
    rng = random.Random(12)
    systems = [random_small_system(rng, max_chains=6, tmax=60) for _ in range(300)]
    systems += [mutate_invalid(random_small_system(rng), rng) for _ in range(100)]
    for flags in (0, 1, 2, 3):
        b = flatten(systems, comm_cost=1, flags=flags)
        _, osch, ost, _ = O.analyze(b)
        b["flags"] = flags | VO
        hb = paam.Batch.from_host(b)
        sets = paam.Sets(hb)
        sched = torch.full((hb.n_sets,), 7, dtype=torch.uint8, device="cuda")
        sets.analyze(None, sched, None)
        torch.cuda.synchronize()
        assert np.array_equal(sched.cpu().numpy(), osch), flags
        sets.free()


def test_verdict_only_rejects_wcrt_output_and_admit_ignores_it():
    p = config3_params()
    n = 20_000
    raw = _raw(p, 6, 0, n, VO)
    sets = paam.Sets(raw)
    wcrt = torch.empty(raw.c.n_chains, dtype=torch.int64, device="cuda")
    with pytest.raises(paam.PaamError):
        sets.analyze(wcrt, None, None)
    with pytest.raises(paam.PaamError):
        sets.pack_analyze(raw, wcrt, None, None)
    # admission names the first failing chain, so it runs the full analysis whatever the flag
    dec_vo = torch.empty(n, dtype=torch.int32, device="cuda")
    sets.admit(dec_vo)
    raw0 = _raw(p, 6, 0, n, 0)
    sets0 = paam.Sets(raw0)
    dec = torch.empty(n, dtype=torch.int32, device="cuda")
    sets0.admit(dec)
    torch.cuda.synchronize()
    assert torch.equal(dec, dec_vo)


@pytest.mark.parametrize("flags", [0, paam.PAAM_FLAG_BLOCKING_SOUND, VO])
def test_sweep_matches_generate_pack_analyze(flags):
    """paam_sweep (device-generated chunks, generation overlapped with analysis, capacity layout) gives
    the verdicts and bins of paam_generate + paam_pack_analyze, over a ragged range of chunks."""
    p = config3_params()
    n, first = 300_001, 12_345
    dev = torch.device("cuda")
    sw = paam.Sweeper(chunk=65_536)
    sched_s = torch.full((n,), 7, dtype=torch.uint8, device=dev)
    bins_s = torch.zeros(2 * p.n_bins, dtype=torch.int64, device=dev)
    sw.run(paam.PaamGenParams.from_buffer_copy(bytes(p)), 4, first, n, sched_s, bins_s, flags=flags)
    sw.run(paam.PaamGenParams.from_buffer_copy(bytes(p)), 4, first, n, None, bins_s, flags=flags)  # reuse: bins x2
    raw = paam.Raw(paam.PaamGenParams.from_buffer_copy(bytes(p)), 4, first, n, flags=flags)
    sets = paam.Sets(raw)
    sched = torch.full((n,), 9, dtype=torch.uint8, device=dev)
    bins = torch.zeros(2 * p.n_bins, dtype=torch.int64, device=dev)
    sets.pack_analyze(raw, None, sched, bins)
    torch.cuda.synchronize()
    assert torch.equal(sched_s, sched)
    assert torch.equal(bins_s, 2 * bins)
    sw.free()
