"""Bit-exact parity of the CUDA path with the CPU oracle on >= 16M synthetic chain sets (the
north_star target): config 4 (config-3 recipe, seed 4), chunks of 1M sets generated on the device,
packed + analysed with paam_pack_analyze, every WCRT / verdict / bin compared with the oracle's own
generate+analyse of the same (seed, index) range on all host cores.

python tools/parity_16m.py [--sets 16000000] [--chunk 1000000]  -> JSON summary on stdout
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from gen.inputs import config3_params
    from oracle import oracle as O
    from paper_2404_06452_b200 import paam

    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", type=int, default=16_000_000)
    ap.add_argument("--chunk", type=int, default=1_000_000)
    ap.add_argument("--seed", type=int, default=4)
    args = ap.parse_args()
    gp = config3_params()
    pp = paam.PaamGenParams.from_buffer_copy(bytes(gp))
    nthreads = os.cpu_count() or 1
    dev = torch.device("cuda")
    tot_bins_g = np.zeros(2 * gp.n_bins, np.int64)
    tot_bins_o = np.zeros(2 * gp.n_bins, np.int64)
    mism_sched = mism_wcrt = 0
    chains = 0
    t_gpu = t_cpu = 0.0
    for first in range(0, args.sets, args.chunk):
        n = min(args.chunk, args.sets - first)
        t0 = time.perf_counter()
        raw = paam.Raw(pp, args.seed, first, n)
        sets = paam.Sets(raw)
        wcrt = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
        sched = torch.empty(n, dtype=torch.uint8, device=dev)
        bins = torch.zeros(2 * gp.n_bins, dtype=torch.int64, device=dev)
        sets.pack_analyze(raw, wcrt, sched, bins)
        torch.cuda.synchronize()
        off = raw.to_host()["set_chain_off"]
        gw = wcrt.cpu().numpy().view(np.uint64)
        gs = sched.cpu().numpy()
        gb = bins.cpu().numpy()
        t_gpu += time.perf_counter() - t0
        sets.free()
        raw.free()
        t0 = time.perf_counter()
        ow, osch, ob, _ = O.generate_analyze(gp, args.seed, first, n, want_wcrt=True, nthreads=nthreads)
        t_cpu += time.perf_counter() - t0
        m = np.diff(off).astype(np.int64)
        idx = np.repeat(np.arange(n, dtype=np.int64), m) * 32 + (np.arange(len(gw), dtype=np.int64) - np.repeat(off[:-1].astype(np.int64), m))
        mism_wcrt += int(np.count_nonzero(gw != ow.reshape(-1)[idx]))
        mism_sched += int(np.count_nonzero(gs != osch))
        tot_bins_g += gb
        tot_bins_o += ob
        chains += len(gw)
        print(f"[{first + n}/{args.sets}] wcrt mismatches {mism_wcrt} sched mismatches {mism_sched}", file=sys.stderr, flush=True)
    out = dict(sets=args.sets, chains=chains, seed=args.seed, workload="config 4 (config-3 recipe)",
               path="paam_pack_analyze on a device batch = fused_kernel (+ wide_kernel for handed-over sets)",
               wcrt_mismatches=mism_wcrt, sched_mismatches=mism_sched,
               bins_equal=bool(np.array_equal(tot_bins_g, tot_bins_o)), bins=tot_bins_g.tolist(),
               schedulable=int(tot_bins_g[1::2].sum()), oracle_threads=nthreads,
               oracle_seconds=round(t_cpu, 1), gpu_path_seconds_incl_copies=round(t_gpu, 1))
    print(json.dumps(out))
    return 0 if (mism_wcrt == 0 and mism_sched == 0 and out["bins_equal"]) else 1


if __name__ == "__main__":
    sys.exit(main())
