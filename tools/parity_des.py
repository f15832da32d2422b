"""DES parity at config-5 size: paam_simulate on 1M config-3-recipe sets (10 s horizon) in the bench's
launch configuration, compared with the oracle DES on a sample of the same sets (blocks of 64 sets
every 1024: 1/16 of the workload) -- per-chain maximum response, completed count, per-set digest --
plus the sim <= bound census over all 1M sets.

python tools/parity_des.py [--sets 1000000] -> JSON on stdout"""
import argparse, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from gen.inputs import config3_params, generate_host
    from oracle import oracle as O
    from paper_2404_06452_b200 import paam
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", type=int, default=1_000_000)
    ap.add_argument("--horizon-s", type=float, default=10.0)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--sim-seed", type=int, default=3)
    ap.add_argument("--block", type=int, default=64)
    ap.add_argument("--every", type=int, default=1024)
    args = ap.parse_args()
    gp = config3_params()
    pp = paam.PaamGenParams.from_buffer_copy(bytes(gp))
    dev = torch.device("cuda")
    n = args.sets
    hz = int(args.horizon_s * 1e9)
    raw = paam.Raw(pp, args.seed, 0, n)
    sets = paam.Sets(raw)
    wcrt = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    sets.analyze(wcrt, None, None)
    resp = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    cnt = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    dig = torch.empty(n, dtype=torch.int64, device=dev)
    viol = torch.zeros(1, dtype=torch.int64, device=dev)
    mis = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    drp = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    sts = torch.empty(n, dtype=torch.int32, device=dev)
    stopped = torch.zeros(1, dtype=torch.int64, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sets.simulate(hz, args.sim_seed, resp, cnt, dig, wcrt, viol, first_index=0, out_misses=mis, out_drops=drp,
                  out_status=sts, out_stopped=stopped)
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1)
    off = raw.to_host()["set_chain_off"]
    g_resp = resp.cpu().numpy().view(np.uint64)
    g_cnt = cnt.cpu().numpy().view(np.uint64)
    g_dig = dig.cpu().numpy().view(np.uint64)
    g_w = wcrt.cpu().numpy().view(np.uint64)
    g_mis = mis.cpu().numpy().view(np.uint64)
    g_drp = drp.cpu().numpy().view(np.uint64)
    g_st = sts.cpu().numpy()
    mism = dict(resp=0, count=0, misses=0, drops=0, digest=0, status=0)
    backlog_sets = 0
    sampled = 0
    t0 = time.perf_counter()
    for first in range(0, n, args.every):
        k = min(args.block, n - first)
        hb = generate_host(gp, args.seed, first, k)
        c0, c1 = int(off[first]), int(off[first + k])
        o = O.simulate(hb, hz, seed=args.sim_seed, first_index=first, bound=g_w[c0:c1], nthreads=os.cpu_count() or 1)
        # D14: a set whose oracle backlog outgrows PAAM_SIM_QCAP slots must be stopped (status BACKLOG) on the
        # device; every other set must agree exactly (statistics per chain, digest, status OK).
        loc = np.diff(off[first:first + k + 1].astype(np.int64))
        set_of_chain = np.repeat(np.arange(k), loc)
        peak = np.zeros(k, np.int64)
        np.maximum.at(peak, set_of_chain, o["peak_live"].astype(np.int64))
        over = peak > paam.PAAM_SIM_QCAP
        backlog_sets += int(over.sum())
        want_st = np.where(over, paam.PAAM_SIM_BACKLOG, paam.PAAM_SIM_OK)
        mism["status"] += int(np.count_nonzero(g_st[first:first + k] != want_st))
        ok_c = ~over[set_of_chain]
        for key, g in (("resp", g_resp), ("count", g_cnt), ("misses", g_mis), ("drops", g_drp)):
            mism[key] += int(np.count_nonzero((o[key] != g[c0:c1]) & ok_c))
        mism["digest"] += int(np.count_nonzero((o["digest"] != g_dig[first:first + k]) & ~over))
        sampled += k
    cpu_s = time.perf_counter() - t0
    out = dict(sets=n, horizon_s=args.horizon_s, sim_seed=args.sim_seed, gpu_ms=round(gpu_ms, 1),
               gpu_sets_per_s=round(n / (gpu_ms / 1e3)), sampled_sets=sampled, mismatches=mism,
               sim_le_bound_violations_all_sets=int(viol.item()),
               stopped_runs_all_sets=int(stopped.item()), backlog_sets_in_sample=backlog_sets,
               misses_all_sets=int(g_mis.sum()), drops_all_sets=int(g_drp.sum()), completed_instances=int(g_cnt.sum()),
               oracle_seconds_for_sample=round(cpu_s, 1), oracle_sets_per_s=round(sampled / cpu_s, 1),
               oracle_threads=os.cpu_count())
    print(json.dumps(out))
    return 0 if sum(mism.values()) == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
