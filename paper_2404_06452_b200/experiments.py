"""Experiments built on the hot path: every number comes from the CUDA kernels
through the C ABI (generate -> pack -> analyze [-> simulate]).

* schedulability curves of the paper's analytical study (Fig. 12): chains per set and the
  accelerator:CPU utilisation ratio swept as generator parameters, ratio of schedulable sets;
* the PAAM_FLAG_BLOCKING_SOUND census (reading A10): simulate shared-executor workloads and count
  sim > bound violations under the paper's blocking term and under the sound variant;
* the PAAM vs FIFO_DIRECT comparison of Case Study 3.
"""
from __future__ import annotations

import numpy as np

from . import paam


def _params(gp) -> paam.PaamGenParams:
    return paam.PaamGenParams.from_buffer_copy(bytes(gp))


def schedulable_ratio(gen_params, seed: int, n: int, comm_cost=100_000, flags=0, first=0, stream=None):
    """Fraction of schedulable sets among n generated sets (GPU)."""
    import torch
    raw = paam.Raw(_params(gen_params), seed, first, n, comm_cost, flags, stream=stream)
    sets = paam.Sets(raw, stream=stream)
    sched = torch.empty(n, dtype=torch.uint8, device="cuda")
    sets.analyze(None, sched, None, stream=stream)
    torch.cuda.synchronize()
    r = int(sched.to(torch.int64).sum().item()) / n
    sets.free()
    raw.free()
    return r


def chain_count_curve(m_values, trials=1000, u_total=0.5, seed=12, **kw):
    """Fig. 12(a): fixed chain length 4, one accelerator, 1:1 ratio; U_total fixed."""
    from gen.inputs import make_params, US
    out = []
    for m in m_values:
        gp = make_params(m_lo=m, m_hi=m, n_bins=1, u_lo=u_total, u_step=0.0,
                         accels=((6, 1, 391 * US, 130 * US),), **kw)
        out.append((m, schedulable_ratio(gp, seed + m, trials)))
    return out


def ratio_curve(ratios=((1, 9), (2, 8), (3, 7), (4, 6), (5, 5), (6, 4), (7, 3)), trials=1000, m=8, u_total=0.5,
                seed=21, **kw):
    """Fig. 12(b): accelerator:CPU utilisation ratio from 1:9 to 7:3."""
    from gen.inputs import make_params, US
    out = []
    for a, c in ratios:
        gp = make_params(m_lo=m, m_hi=m, n_bins=1, u_lo=u_total, u_step=0.0, ratio_acc=a, ratio_cpu=c,
                         accels=((6, 1, 391 * US, 130 * US),), **kw)
        out.append((f"{a}:{c}", schedulable_ratio(gp, seed, trials)))
    return out


def blocking_census(gen_params, seed: int, n: int, horizon_ns: int, sim_seed: int = 1, comm_cost=100_000):
    """Simulate n sets; count violations of the as-written and of the sound bound (A10)."""
    import torch
    res = {}
    for name, flags in (("as_written", 0), ("sound", paam.PAAM_FLAG_BLOCKING_SOUND)):
        raw = paam.Raw(_params(gen_params), seed, 0, n, comm_cost, flags)
        sets = paam.Sets(raw)
        wcrt = torch.empty(raw.c.n_chains, dtype=torch.int64, device="cuda")
        sched = torch.empty(n, dtype=torch.uint8, device="cuda")
        sets.analyze(wcrt, sched, None)
        resp = torch.empty(raw.c.n_chains, dtype=torch.int64, device="cuda")
        viol = torch.zeros(1, dtype=torch.int64, device="cuda")
        sets.simulate(horizon_ns, sim_seed, resp, None, None, wcrt, viol)
        torch.cuda.synchronize()
        res[name] = {"schedulable_sets": int(sched.sum().item()), "violating_chains": int(viol.item())}
        sets.free()
        raw.free()
    return res


def fifo_comparison(batch_dict, horizon_ns: int, seeds=range(8)):
    """Max observed response per chain under PAAM and under FIFO_DIRECT (GPU), over several phasings."""
    import torch
    hb = paam.Batch.from_host(batch_dict)
    sets = paam.Sets(hb)
    nch = hb.c.n_chains
    wcrt = torch.empty(nch, dtype=torch.int64, device="cuda")
    sets.analyze(wcrt, None, None)
    best = {"paam": np.zeros(nch, np.uint64), "fifo": np.zeros(nch, np.uint64)}
    for sd in seeds:
        for mode in ("paam", "fifo"):
            resp = torch.empty(nch, dtype=torch.int64, device="cuda")
            sets.simulate(horizon_ns, sd, resp, fifo=(mode == "fifo"))
            torch.cuda.synchronize()
            best[mode] = np.maximum(best[mode], resp.cpu().numpy().view(np.uint64))
    best["bound"] = wcrt.cpu().numpy().view(np.uint64)
    sets.free()
    return best
