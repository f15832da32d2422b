#!/usr/bin/env python
"""bench.py -- chain sets analysed per second (PAAM WCRT fixed points) on N B200s.

One step = the whole hot path over this rank's batch of synthetic chain sets that is already
resident in HBM: paam_pack_analyze = one fused_kernel launch (validate + derive, §8(a) step 2, then
the Lemma 2 / Eq.5 fixed points, end-to-end WCRT, verdict and bin counts of steps 3-6, the derived
records kept on chip) -> (N > 1) one NCCL all-reduce of the bin counts.  Weak scaling: every rank owns SETS_PER_GPU consecutive set indices of
the config-4 stream (seed 4), so N = 8 is exactly config 4 (16M sets) and N = 1 is the config-3
recipe on 2M sets.

Extra legs in the same JSON line: the kernel's per-launch time (roofline: HBM, issue and ALU views),
the split entry points (paam_repack + paam_analyze) for reference, verdict_only (PAAM_FLAG_VERDICT_ONLY),
e2e (the same metric from pinned host buffers through paam_pack_analyze32 -- the compact batch, 32-bit
times and one byte per segment -- with every WCRT copied back, H2D / D2H inside the timed region),
e2e_u64 (the same through paam_pack_analyze on the u64 batch), e2e_verdict_only, e2e_device_generate
(paam_sweep: device generation included), des (config-5 leg: paam_simulate on 1M sets, 10 s horizon, sim <= bound
census, misses / drops / stopped runs, with and without digests), cpu_baseline (the oracle).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0 (the driver's contract).  The CPU oracle is executed only by the
cpu_baseline leg (rank 0, N = 1) and by --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "chain-sets analysed/sec (WCRT fixed-point) at 1/2/4/8 B200; % of roofline"
SEED = 4
DEFAULT_SETS_PER_GPU = 2_000_000
# Algorithmic integer work of one mu-term of Eq.2-Eq.5 after exact regrouping: multiply-high by the
# period's magic constant, shift, multiply by the interfering weight, accumulate.
OPS_PER_MU = 4


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # one process per GPU over NCCL; PAAM_DIST_BACKEND=gloo runs the same N > 1 path over gloo (CUDA
        # tensors, host staging), e.g. several ranks on one GPU in the multi-process test
        backend = os.environ.get("PAAM_DIST_BACKEND", "nccl")
        dev = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline(params, first, budget_s=15.0, nthreads=None):
    """The oracle as it stands, on a bounded prefix of this rank's workload, all host cores.
    The sample is generated first (untimed); only the oracle's analysis is timed."""
    from gen.inputs import generate_host
    from oracle import oracle as O
    nthreads = nthreads or (os.cpu_count() or 1)
    probe = generate_host(params, SEED, first, 2000)
    t0 = time.perf_counter()
    O.analyze(probe, nthreads=nthreads)
    rate = 2000 / max(time.perf_counter() - t0, 1e-6)
    n = int(min(max(rate * budget_s, 2000), 2_000_000))
    sample = generate_host(params, SEED, first, n)
    t0 = time.perf_counter()
    O.analyze(sample, nthreads=nthreads)
    dt = time.perf_counter() - t0
    n1 = max(500, min(n, int(n / nthreads / 4)))  # one thread, about a quarter of the budget
    one = generate_host(params, SEED, first, n1)
    t1 = time.perf_counter()
    O.analyze(one, nthreads=1)
    dt1 = time.perf_counter() - t1
    return {"value": n / dt, "unit": "chain-sets/s", "cores": nthreads, "kind": "oracle",
            "value_1_thread": n1 / dt1,
            "sample": f"first {n} sets of this rank's range (config-3 recipe, seed {SEED}): {dt:.1f} s "
                      f"of oracle analysis on {nthreads} threads; 1 thread: first {n1} sets, {dt1:.1f} s"}


def run_reference(args):
    """--impl reference: the CPU oracle timed as it stands (this tier's reference arm)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from gen.inputs import config3_params, generate_host
    from oracle import oracle as O
    p = config3_params()
    nthreads = os.cpu_count() or 1
    per_step = args.ref_sets_per_step
    batches = [generate_host(p, SEED, i * per_step, per_step) for i in range(args.warmup + args.steps)]
    for i in range(args.warmup):
        O.analyze(batches[i], nthreads=nthreads)
    t0 = time.perf_counter()
    for i in range(args.steps):
        O.analyze(batches[args.warmup + i], nthreads=nthreads)
    dt = time.perf_counter() - t0
    v = per_step * args.steps / dt
    out = {"metric": METRIC, "value": v, "unit": "chain-sets/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": workload_name(args.sets_per_gpu), "sets_per_gpu": args.sets_per_gpu,
                      "global_sets": world * args.sets_per_gpu, "seed": SEED,
                      "reference_sample": f"each step analyses {per_step} sets of that workload (bounded so the "
                                          f"run ends within minutes); value is sets/s over the sampled sets"},
           "cpu_baseline": {"value": v, "unit": "chain-sets/s", "cores": nthreads, "kind": "oracle",
                            "sample": f"{per_step} sets per step x {args.steps} steps"},
           "e2e": {"value": v, "unit": "chain-sets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def workload_name(n: int) -> str:
    """The bench workload (both arms): config-3 recipe, n sets per GPU, set-index shards."""
    return (f"config-3 recipe (m 8-16 chains x 4 callbacks, GPU-like n=6 + TPU-like n=1, 9 utilisation bins), "
            f"{n} sets/GPU, seed {SEED}, rank r owns [r*{n}, (r+1)*{n}) -- N=8 is config 4 (16M sets)")


def batch32_bytes(b32) -> int:
    return int(sum(a.nbytes for k, a in b32.arrays.items() if a is not None and not k.endswith("_pinned")))


def batch_bytes(c) -> int:
    n, ch, cb, sg, ex, ac = c.n_sets, c.n_chains, c.n_cbs, c.n_segs, c.n_execs, c.n_accels
    return (3 * 4 * (n + 1) + ch * (8 + 8 + 4 + 1) + 4 * (ch + 1) + cb * 2 + 4 * (cb + 1) + sg * (1 + 8 + 1 + 1)
            + ex * (1 + 4 + 1) + ac * (1 + 1 + 1 + 8 + 8) + (4 * n if c.set_bin else 0))


def run_ours(args):
    import numpy as np
    import torch
    from paper_2404_06452_b200 import paam

    world, rank, local = dist_setup(args.gpus)
    dev = torch.device("cuda", torch.cuda.current_device())
    from paper_2404_06452_b200.shard import allreduce_bins, shard_range
    first, n = shard_range(rank, world, args.sets_per_gpu)
    from gen.inputs import config3_params  # workload recipe (shared input generator params)
    gp = config3_params()
    params = paam.PaamGenParams.from_buffer_copy(bytes(gp))
    stream = torch.cuda.Stream(device=dev)

    # ---- inputs resident in HBM (generated on device; outside the timed region) ------------------
    with torch.cuda.stream(stream):
        raw = paam.Raw(params, SEED, first, n, stream=stream)
        sets = paam.Sets(raw, stream=stream)
        wcrt = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
        sched = torch.empty(n, dtype=torch.uint8, device=dev)
        bins = torch.zeros(2 * gp.n_bins, dtype=torch.int64, device=dev)
    stream.synchronize()
    rec_bytes = paam.lib().paam_record_bytes()
    in_bytes = batch_bytes(raw.c)

    dist = None
    if world > 1:
        import torch.distributed as dist

    def step():
        # §8(a) steps 2-6 pipelined: pack_kernel of chunk i+1 overlaps analyze_kernel of chunk i
        sets.pack_analyze(raw, wcrt, sched, bins, stream=stream)
        if dist is not None:                                  # the one exchange: bin counts
            allreduce_bins(bins, stream=stream)

    # ---- warm-up ------------------------------------------------------------------------------------
    for _ in range(args.warmup):
        step()
    stream.synchronize()
    barrier(world)

    # ---- timed region: K steps, CUDA events on the launching stream ---------------------------------
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = paam.kernel_launches()
    torch.cuda.synchronize()
    barrier(world)
    start.record(stream)
    for k in range(args.steps):
        step()
    end.record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    launches = paam.kernel_launches() - launches0
    clk = clocks.stop()
    ms_local = start.elapsed_time(end)
    ms = max_over_ranks(ms_local, world)
    value = world * n * args.steps / (ms / 1e3)

    # ---- the timed kernel's launch durations: CUDA events around each launch on `stream` -----------
    # (one fused_kernel launch per step: paam_pack_analyze on a device-resident batch)
    kev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    for k in range(args.steps):
        kev[k][0].record(stream)
        sets.pack_analyze(raw, wcrt, sched, bins, stream=stream)
        kev[k][1].record(stream)
    stream.synchronize()
    fused_ms = [e[0].elapsed_time(e[1]) for e in kev]
    # the split entry points (paam_repack -> paam_analyze: pack_kernel writes records, analyze_kernel
    # reads them), timed the same way for reference
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    for k in range(args.steps):
        ev[k][0].record(stream)
        sets.repack(raw, stream=stream)
        ev[k][1].record(stream)
        sets.analyze(wcrt, sched, bins, stream=stream)
        ev[k][2].record(stream)
    stream.synchronize()
    pack_ms = [e[0].elapsed_time(e[1]) for e in ev]
    ana_ms = [e[1].elapsed_time(e[2]) for e in ev]
    with torch.cuda.stream(stream):
        bins.zero_()  # on the kernel's stream (a default-stream zero could race the kernel)
    sets.pack_analyze(raw, wcrt, sched, bins, stream=stream)  # one clean pass for the reported bin counts
    if dist is not None:
        allreduce_bins(bins, stream=stream)
    stream.synchronize()

    # ---- verdict-only sweep mode (PAAM_FLAG_VERDICT_ONLY: no WCRTs, early exit at the first miss) ----
    import types
    vb = paam.PaamBatch.from_buffer_copy(raw.c)
    vb.flags |= paam.PAAM_FLAG_VERDICT_ONLY
    vbatch = types.SimpleNamespace(c=vb)
    vbins = torch.zeros_like(bins)
    stream.wait_stream(torch.cuda.current_stream())  # the allocations / zeroing above precede the kernels
    for _ in range(args.warmup):
        sets.pack_analyze(vbatch, None, sched, vbins, stream=stream)
    stream.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        sets.pack_analyze(vbatch, None, sched, vbins, stream=stream)
        if dist is not None:
            allreduce_bins(vbins, stream=stream)
    e1.record(stream)
    stream.synchronize()
    vo_ms = max_over_ranks(e0.elapsed_time(e1), world)
    verdict_only = {"value": world * n * args.steps / (vo_ms / 1e3), "unit": "chain-sets/s",
                    "ms_per_step": vo_ms / args.steps,
                    "note": "paam_pack_analyze with PAAM_FLAG_VERDICT_ONLY: verdicts + bins only, analysis of a "
                            "set stops at its first CRITICAL deadline miss"}

    # ---- e2e including device generation: paam_sweep (generate -> pack -> analyze, chunked, generation
    # overlapped with analysis) -> D2H of the verdicts and bins -----------------------------------------
    e2e_gen = None
    if not args.no_e2e:
        sched_g = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        bins_g = torch.empty(2 * gp.n_bins, dtype=torch.int64, pin_memory=True)
        gbins = torch.zeros_like(bins)
        stream.wait_stream(torch.cuda.current_stream())
        sweeper = paam.Sweeper()

        def gen_step():
            with torch.cuda.stream(stream):
                gbins.zero_()
            sweeper.run(params, SEED, first, n, sched, gbins, stream=stream)
            if dist is not None:
                allreduce_bins(gbins, stream=stream)
            with torch.cuda.stream(stream):
                sched_g.copy_(sched, non_blocking=True)
                bins_g.copy_(gbins, non_blocking=True)
            stream.synchronize()
        for _ in range(max(1, args.warmup)):
            gen_step()
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            gen_step()
        gen_s = max_over_ranks(time.perf_counter() - t0, world)
        e2e_gen = {"value": world * n * args.steps / gen_s, "unit": "chain-sets/s", "ms_per_step": 1e3 * gen_s / args.steps,
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": n + 8 * 2 * gp.n_bins,
                   "note": "host wall clock per step: paam_sweep (device generation of 256k-set chunks overlapped "
                           "with pack + analyze of the previous chunk) + D2H of verdicts and bins"}
        if sum(bins_g.tolist()[0::2]) != world * n:
            raise RuntimeError("paam_sweep bin totals do not match the sets")
        sweeper.free()
    sets.pack_analyze(raw, wcrt, sched, vbins, stream=stream)  # the handle again describes `raw` (DES leg)
    stream.synchronize()

    # ---- e2e: the same metric through the C ABI with HOST buffers (copies inside the region) ------
    # Each step copies the pinned host batch in (chunked, overlapped with the kernel of earlier chunks)
    # and reads every WCRT, verdict and the bin counts back: the full output of the timed step.
    e2e = e2e_vo = e2e_u64 = None
    if not args.no_e2e:
        from gen.inputs import generate_host

        def pinned(nbytes):
            return torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True).numpy()

        host = generate_host(gp, SEED, first, n, pinned_alloc=pinned)
        hb = paam.Batch.from_host(host)
        hvb = paam.Batch.from_host(dict(host, flags=paam.PAAM_FLAG_VERDICT_ONLY))
        wcrt_h = torch.empty(hb.c.n_chains, dtype=torch.int64, pin_memory=True)
        sched_h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        bins_h = torch.empty(2 * gp.n_bins, dtype=torch.int64, pin_memory=True)
        hsets = paam.Sets(hb, stream=stream)
        ebins = torch.zeros_like(bins)
        stream.wait_stream(torch.cuda.current_stream())

        def e2e_step(batch, with_wcrt):
            with torch.cuda.stream(stream):
                ebins.zero_()
            # host outputs: the library copies every chunk's WCRTs and verdicts back into these pinned
            # buffers as soon as the chunk is analysed (overlapping the next chunk's H2D)
            hsets.pack_analyze(batch, wcrt_h if with_wcrt else None, sched_h, ebins, stream=stream)
            if dist is not None:
                allreduce_bins(ebins, stream=stream)
            with torch.cuda.stream(stream):
                bins_h.copy_(ebins, non_blocking=True)  # D2H: the bin counts
            stream.synchronize()

        def timed(batch, with_wcrt):
            for _ in range(max(1, args.warmup)):
                e2e_step(batch, with_wcrt)
            barrier(world)
            t0 = time.perf_counter()
            for _ in range(args.steps):
                e2e_step(batch, with_wcrt)
            return max_over_ranks(time.perf_counter() - t0, world)
        ref_w = wcrt.cpu().numpy()
        d2h_full = 8 * hb.c.n_chains + n + 8 * 2 * gp.n_bins
        u64_s = timed(hb, True)
        if not np.array_equal(wcrt_h.numpy(), ref_w):
            raise RuntimeError("e2e (u64 batch) WCRTs differ from the device-resident run")
        e2e_u64 = {"value": world * n * args.steps / u64_s, "unit": "chain-sets/s",
                   "h2d_bytes_per_step": batch_bytes(hb.c), "d2h_bytes_per_step": d2h_full,
                   "ms_per_step": 1e3 * u64_s / args.steps,
                   "note": "paam_pack_analyze from pinned host buffers (u64 CSR batch, chunked H2D overlapped with "
                           "the kernel) + D2H of every WCRT, verdict and bin count; host wall clock, max over ranks"}
        # the compact batch (paam_batch32: the same sets in 32-bit times and one byte per segment), pinned
        hb32 = paam.Batch32.from_host(host, pin=True)
        hvb32 = paam.Batch32.from_host(dict(host, flags=paam.PAAM_FLAG_VERDICT_ONLY), pin=True)
        wcrt_h.zero_()
        e2e_s = timed(hb32, True)
        if not np.array_equal(wcrt_h.numpy(), ref_w):
            raise RuntimeError("e2e (compact batch) WCRTs differ from the device-resident run")
        e2e = {"value": world * n * args.steps / e2e_s, "unit": "chain-sets/s",
               "h2d_bytes_per_step": batch32_bytes(hb32), "d2h_bytes_per_step": d2h_full,
               "ms_per_step": 1e3 * e2e_s / args.steps,
               "note": "paam_pack_analyze32 from pinned host buffers (the compact batch: 32-bit times, one byte per "
                       "segment; chunked H2D overlapped with the kernel) into pinned host outputs (every WCRT and "
                       "verdict, copied back per chunk) + D2H of the bin counts; "
                       "host wall clock, max over ranks.  e2e_u64: the same through the u64 batch"}
        vo_s = timed(hvb32, False)
        e2e_vo = {"value": world * n * args.steps / vo_s, "unit": "chain-sets/s",
                  "h2d_bytes_per_step": batch32_bytes(hb32), "d2h_bytes_per_step": n + 8 * 2 * gp.n_bins,
                  "ms_per_step": 1e3 * vo_s / args.steps,
                  "note": "as e2e with PAAM_FLAG_VERDICT_ONLY: verdicts and bins only"}
        hsets.free()
    sets.pack_analyze(raw, wcrt, sched, vbins, stream=stream)  # the handle again describes `raw` (DES leg)
    stream.synchronize()

    # ---- config 5 leg: the paired DES (paam_simulate) with the sim <= bound census -------------------
    des = None
    if args.des_sets > 0:
        nd = min(args.des_sets, n)
        z = lambda k: torch.zeros(k, dtype=torch.int64, device=dev)
        resp, cnt, miss, drop = (z(raw.c.n_chains) for _ in range(4))
        dig, viol, stopped = z(n), z(1), z(1)
        status = torch.empty(n, dtype=torch.int32, device=dev)
        wit = torch.full((2 * 64,), -1, dtype=torch.int32, device=dev)
        hz = int(args.des_horizon_s * 1e9)
        stream.wait_stream(torch.cuda.current_stream())  # the zeroed outputs precede the kernels
        sets.simulate(hz, 3, resp, None, dig, None, None, first_index=first, n=min(nd, 1024), stream=stream)  # warm-up
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = paam.kernel_launches()
        e0.record(stream)
        sets.simulate(hz, 3, resp, cnt, dig, wcrt, viol, first_index=first, n=nd, stream=stream, out_misses=miss,
                      out_drops=drop, out_status=status, out_witness=wit, out_stopped=stopped)
        e1.record(stream)
        stream.synchronize()
        des_ms = max_over_ranks(e0.elapsed_time(e1), world)
        des_launches = paam.kernel_launches() - l0
        tot = torch.stack([viol[0], stopped[0], cnt.sum(), miss.sum(), drop.sum()]).clone()
        e0.record(stream)  # the same simulation without event digests (out_digest = NULL)
        sets.simulate(hz, 3, resp, None, None, wcrt, None, first_index=first, n=nd, stream=stream)
        e1.record(stream)
        stream.synchronize()
        des_nd_ms = max_over_ranks(e0.elapsed_time(e1), world)
        if dist is not None:
            dist.all_reduce(tot)
        tot = tot.tolist()
        des = {"metric": "chain-sets simulated/sec (PAAM DES, config-5 leg)", "value": world * nd / (des_ms / 1e3),
               "unit": "chain-sets/s", "sets_per_gpu": nd, "horizon_s": args.des_horizon_s, "seed": 3,
               "ms": des_ms, "digests": True, "value_without_digests": world * nd / (des_nd_ms / 1e3),
               "sim_le_bound_violations": int(tot[0]), "stopped_sets": int(tot[1]),
               "completed_instances": int(tot[2]), "deadline_misses": int(tot[3]), "be_drops": int(tot[4]),
               "gpu_launches": des_launches,
               "scope": "violations counted in the sets the analysis declares schedulable (every CRITICAL chain "
                        "R* <= D) whose run was not stopped; stopped_sets = runs stopped by PAAM_SIM_BACKLOG / STEPCAP"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    case_studies = case_study_leg(paam, torch, dev) if not args.no_case_studies else None

    # ---- roofline of the timed kernel ---------------------------------------------------------------
    # fused_kernel is the whole step.  Algorithmic bytes per launch: the raw CSR batch it must read
    # (§8(b) paam_batch) + the outputs it must write (u64 WCRT per chain, u8 verdict per set, bins).
    pk = peaks()
    hbm_peak = pk.get("hbm_gbs", 6533.2)
    clk_ghz = (clk.get("sm_mhz") or 1965.0) / 1e3
    fused_avg = sum(fused_ms) / len(fused_ms)
    traffic = measured_traffic_per_set()
    issue = ncu_issue_stats()
    out_bytes = 8 * raw.c.n_chains + n + 16 * gp.n_bins
    alg_bytes = in_bytes + out_bytes
    roof = {"bound": "hbm", "achieved": alg_bytes / (fused_avg / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": alg_bytes / (fused_avg / 1e3) / 1e9 / hbm_peak,
            "traffic": None if not traffic or "fused_kernel" not in traffic else traffic["fused_kernel"] * n,
            "kernel": "fused_kernel", "kernel_ms": fused_avg, "share_of_step": fused_avg / (ms / args.steps),
            "algorithmic_bytes": alg_bytes, "bytes_per_set": alg_bytes / n,
            "peak_of": "measured (MEASURED_PEAKS.json hbm_gbs)" if pk else "fallback (B200_PROFILING.md)",
            "ncu_issue": issue.get("fused_kernel"),
            "note": "two launches per step, fused_kernel and wide_kernel (whose list is empty for config 3); per-launch CUDA events on the bench stream. The kernel is issue-bound "
                    "(see issue): its HBM traffic is the raw batch once, the derived records stay on chip"}
    # issue roofline: warp-instructions per set (ncu) x sets/s vs 148 SMs x 4 schedulers x clock
    iss = issue.get("fused_kernel") or {}
    if iss.get("warp_inst_per_set"):
        ach = iss["warp_inst_per_set"] * n / (fused_avg / 1e3) / 1e12
        peak_issue = 148 * 4 * clk_ghz / 1e3
        roof["issue"] = {"achieved": ach, "peak": peak_issue, "unit": "T warp-instructions/s", "frac": ach / peak_issue,
                         "warp_inst_per_set": iss["warp_inst_per_set"]}
    # the algorithmic integer work (oracle-counted regrouped mu-terms x 4 ops) against the ALU roof
    work = work_per_set(gp, first)
    alu_peak = 148 * 128 * clk_ghz / 1e3  # T lane-ops/s: 148 SMs x 128 int32 lanes/clk (alu + fma pipes)
    ops = work["mu_regrouped_per_set"] * OPS_PER_MU * n
    other = {"bound": "alu", "achieved": ops / (fused_avg / 1e3) / 1e12, "peak": alu_peak,
             "unit": "Tops/s (int32 lane-ops)", "frac": ops / (fused_avg / 1e3) / 1e12 / alu_peak,
             "kernel": "fused_kernel", "ops_per_set": work["mu_regrouped_per_set"] * OPS_PER_MU,
             "peak_source": "derived: 148 SMs x 128 int32 lanes/clk (B300_MICROARCH alu+fma pipes) x measured SM clock"}
    split = {"pack_kernel_ms": sum(pack_ms) / len(pack_ms), "analyze_kernel_ms": sum(ana_ms) / len(ana_ms),
             "note": "paam_repack + paam_analyze (records written to / read from HBM), same batch, for reference",
             "ncu": {k: issue.get(k) for k in ("pack_kernel", "analyze_kernel")},
             "dram_bytes_per_set": {k: (traffic or {}).get(k) for k in ("pack_kernel", "analyze_kernel")}}
    if des is not None:
        di = issue.get("simulate_kernel") or {}
        if di.get("warp_inst_per_set"):
            ach = di["warp_inst_per_set"] * des["value"] / world / 1e12
            peak_issue = 148 * 4 * clk_ghz / 1e3
            des["roofline"] = {"bound": "alu", "achieved": ach, "peak": peak_issue, "unit": "T warp-instructions/s",
                               "frac": ach / peak_issue, "traffic": None if not traffic or "simulate_kernel" not in traffic
                               else traffic["simulate_kernel"] * nd,
                               "kernel": "simulate_kernel", "warp_inst_per_set": di["warp_inst_per_set"],
                               "note": "issue roofline: the DES state lives in shared memory (DRAM traffic is the raw "
                                       "batch and the outputs); warp-instructions per set from the committed ncu capture"}
    out = {"metric": METRIC, "value": value, "unit": "chain-sets/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u32", "data": "synthetic",
           "config": {"workload": workload_name(n), "sets_per_gpu": n, "global_sets": world * n, "seed": SEED,
                      "l2": f"inputs larger than L2: the {in_bytes / 1e9:.1f} GB raw batch is read once per step",
                      "parallelism": f"dp{world} (set-index shards, NCCL all-reduce of bin counts)"},
           "gpu_launches": int(launches), "clocks": clk, "roofline": roof, "roofline_alu": other,
           "split_path": split, "bins": bins.cpu().tolist()}
    if e2e:
        out["e2e"] = e2e
        out["e2e_u64"] = e2e_u64
        out["e2e_verdict_only"] = e2e_vo
    if e2e_gen:
        out["e2e_device_generate"] = e2e_gen
    out["verdict_only"] = verdict_only
    if case_studies:
        out["case_studies"] = case_studies
    if des:
        out["des"] = des
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(gp, first, budget_s=args.cpu_budget)
    if sum(out["bins"][0::2]) != world * n:
        raise RuntimeError(f"bin totals {sum(out['bins'][0::2])} != sets {world * n}")
    print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def case_study_leg(paam, torch, dev, phasings=256, horizon_ms=3000):
    """Configs 1a / 1b: the paper's Case Study 3 (n = 6 and n = 1) and the Case-Study-1
    shaped set (invented numbers, gen/inputs.CS1_SHAPED) through the fused path, and the DES over
    `phasings` release phasings (the set replicated, phases from (seed, set index)) in PAAM mode and in
    the FIFO_DIRECT baseline the paper compares against."""
    import numpy as np
    from gen.inputs import MS, US, case_study_1_shaped, case_study_3, flatten
    out = {}
    for name, s in (("cs3_n6", case_study_3(6)), ("cs3_n1", case_study_3(1)), ("cs1_shaped", case_study_1_shaped())):
        b = flatten([s] * phasings, comm_cost=100 * US)
        wcrt, sched, status, _ = paam.analyze(paam.Batch.from_host(b), fused=True)
        m = len(s.chains)
        hb = paam.Batch.from_host(b)
        sets = paam.Sets(hb)
        bound = torch.from_numpy(wcrt.view(np.int64).copy()).to(dev)
        res = {}
        for mode in ("paam", "fifo_direct"):
            resp = torch.zeros(hb.c.n_chains, dtype=torch.int64, device=dev)
            viol = torch.zeros(1, dtype=torch.int64, device=dev)
            st = torch.empty(phasings, dtype=torch.int32, device=dev)
            sets.simulate(horizon_ms * MS, 1, resp, bound=bound, out_violations=viol, out_status=st,
                          fifo=(mode == "fifo_direct"))
            torch.cuda.synchronize()
            r = resp.cpu().numpy().view(np.uint64).reshape(phasings, m)
            res[mode] = {"max_observed_ms": [round(float(x) / 1e6, 3) for x in r.max(axis=0)],
                         "violations": int(viol.item()), "stopped_runs": int((st.cpu().numpy() != 0).sum())}
            if res[mode]["stopped_runs"]:
                res[mode]["note"] = ("runs stopped by PAAM_SIM_BACKLOG (a CRITICAL chain's backlog outgrew the device's "
                                     "instance slots, D14): their maxima cover the exact prefix, lower bounds")
        sets.free()
        w = wcrt[:m]
        out[name] = {"schedulable": bool(sched[0]),
                     "critical": [ch.cls == 0 for ch in s.chains],
                     "wcrt_bound_ms": [None if x == paam.UNSCHED else round(float(x) / 1e6, 3) for x in w],
                     "des_paam": res["paam"], "des_fifo_direct": res["fifo_direct"],
                     "phasings": phasings, "horizon_ms": horizon_ms}
    out["note"] = ("configs 1a (Case Study 3, PAPER.md:971-974) and 1b (Case Study 1's shape, PAPER.md:488-499, "
                   "invented numbers); bounds from the fused kernel, DES maxima over the phasings; the DES of "
                   "BE chains is unbounded by the analysis (their bound is UNSCHED)")
    return out


def work_per_set(gp, first, sample=4000):
    """Oracle-counted mu-terms per set on a sample of the workload (algorithmic work, not timing)."""
    try:
        from oracle import oracle as O
        _, _, _, cnt = O.generate_analyze(gp, SEED, first, sample, nthreads=os.cpu_count() or 1)
        return {"mu_literal_per_set": float(cnt[0]) / sample, "mu_regrouped_per_set": float(cnt[1]) / sample,
                "iterations_per_set": float(cnt[2]) / sample}
    except Exception:
        return {"mu_literal_per_set": None, "mu_regrouped_per_set": 780.0, "iterations_per_set": None}


def measured_traffic_per_set():
    """DRAM bytes per set of each kernel from the committed ncu --set full capture, if present."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return {k: float(v["dram_bytes_per_set"]) for k, v in d.items() if not k.startswith("_")}
    except Exception:
        return None


def ncu_issue_stats():
    """Issue-slot utilisation and warp instructions per set of each kernel (same committed capture)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return {k: {"issue_active_pct": v.get("issue_active_pct"), "warp_inst_per_set": v.get("warp_inst_per_set"),
                    "source": v.get("source", "profiles/traffic.json (ncu --set full, profiles/r01_ncu_full_v15_summary.txt)")}
                for k, v in d.items() if not k.startswith("_")}
    except Exception:
        return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sets-per-gpu", type=int, default=DEFAULT_SETS_PER_GPU)
    ap.add_argument("--ref-sets-per-step", type=int, default=20_000)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-case-studies", action="store_true")
    ap.add_argument("--des-sets", type=int, default=1_000_000, help="sets per GPU for the DES leg (config 5: 1M; 0 = skip)")
    ap.add_argument("--des-horizon-s", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 untimed warm-up steps
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
