"""GPU parity: the CUDA path (through the C ABI) is bit-exact with the CPU oracle.

Integer results -> bit-exact comparison of every WCRT, verdict, status and bin count.
"""
import json
import os
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen.inputs import (CRITICAL, MS, US, Seg, System, acc, cb, config2_params, config3_params, cpu, flatten,
                        generate_host, make_params, slice_sets)
from oracle import oracle as O
from paper_2404_06452_b200 import paam
from tests.ref_scan import random_small_system
from gen.inputs import case_study_1_shaped
from tests.test_oracle_pins import GOLD, a10_system, app_b_two_chains, cs3_system, two_chain_accel_system

NPROC = os.cpu_count() or 1


def gpu_host_path(batch):
    return paam.analyze(paam.Batch.from_host(batch))


def gpu_device_path(batch):
    return paam.analyze(paam.Batch.from_host_to_device(batch))


def assert_same(batch, gpu, fused_too=True):
    """The given GPU result (split path: paam_pack + paam_analyze) and the fused path (paam_pack_analyze,
    fused_kernel, host batch) against the oracle, element by element."""
    ow, osch, ost, ob = O.analyze(batch, nthreads=NPROC)
    results = [("split", gpu)]
    if fused_too:
        results.append(("fused", paam.analyze(paam.Batch.from_host(batch), fused=True)))
    for name, (gw, gsch, gst, gb) in results:
        assert np.array_equal(ost, gst), (name, np.nonzero(ost != gst)[0][:10])
        bad = np.nonzero(ow != gw)[0]
        assert bad.size == 0, (name, bad[:10], ow[bad[:10]], gw[bad[:10]])
        assert np.array_equal(osch, gsch), name
        if batch.get("n_bins"):
            assert np.array_equal(ob, gb), name


def test_worked_examples_on_gpu():
    systems = [two_chain_accel_system(), two_chain_accel_system(eps=391 * US), app_b_two_chains(),
               cs3_system(6), cs3_system(1), a10_system(), case_study_1_shaped()]  # + config 1b
    for flags in (0, 1):
        b = flatten(systems, comm_cost=0, flags=flags)
        assert_same(b, gpu_host_path(b))
    gw, gsch, _, _ = gpu_host_path(flatten([cs3_system(6)], comm_cost=0))
    assert gw[:2].tolist() == GOLD["cs3_n6"]["R"]
    gw, _, _, _ = gpu_host_path(flatten([app_b_two_chains()], comm_cost=0))
    assert gw.tolist() == GOLD["two_chains_one_executor"]["R"]


@pytest.mark.parametrize("flags", [0, 1])
def test_random_small_systems(flags):
    rng = random.Random(77 + flags)
    systems = [random_small_system(rng, max_chains=6, tmax=200) for _ in range(3000)]
    b = flatten(systems, comm_cost=3, flags=flags)
    assert_same(b, gpu_host_path(b))
    assert_same(b, gpu_device_path(b))


def mutate_invalid(s: System, rng):
    """Break one validation rule (or none)."""
    k = rng.randrange(11)
    if k == 0 and len(s.chains) > 1:
        s.chains[1].prio = s.chains[0].prio
    elif k == 1:
        s.chains[0].D = s.chains[0].T + 1
        s.chains[0].cls = CRITICAL
    elif k == 2:
        s.chains[0].cbs[0].exec = 31
    elif k == 3:
        s.chains[0].cbs[0].segs.append(Seg(1, 1, 3, 0))
    elif k == 4:
        s.chains[0].cbs[0].segs[0].wcet = 0
    elif k == 5:
        s.execs[0] = (10, 1, 0)  # server core of accelerator 0
    elif k == 6:
        s.chains[0].T = 1 << 48
    elif k == 7:
        s.chains[0].cbs[0].segs.append(Seg(s.chains[0].cbs[0].segs[-1].kind, 1))
    elif k == 8 and len(s.execs) > 1:
        s.execs[1] = (s.execs[0][0], s.execs[0][1], s.execs[1][2])  # same core, same process priority
    return s


def test_validation_statuses_match():
    rng = random.Random(5)
    systems = [mutate_invalid(random_small_system(rng), rng) for _ in range(2000)]
    b = flatten(systems, comm_cost=1)
    _, _, st, _ = O.analyze(b)
    assert len(set(st.tolist())) >= 6
    assert_same(b, gpu_host_path(b))


def test_edge_cases():
    # empty set, single chain, maximum sizes: 32 chains, 64 accelerator segments over 8 units
    s0 = System(); s0.accel(server_core=0)
    s1 = System(); a = s1.accel(server_core=0); x = s1.executor(core=1)
    s1.chain(T=10, prio=1, cbs=[cb(x, acc(a, 3))])
    big = System()
    accs = [big.accel(buckets=6, units=2, server_core=20, eps=2, kappa=1),
            big.accel(buckets=1, units=2, server_core=21, eps=1),
            big.accel(buckets=3, units=2, server_core=22),
            big.accel(buckets=2, units=2, server_core=23)]
    xs = [big.executor(core=i % 4, prio=i // 4 + 1) for i in range(16)]
    rng = random.Random(3)
    for c in range(32):
        cbs = []
        for j in range(2):
            aa = accs[(c + j) % 4]
            cbs.append(cb(xs[c % 16], cpu(rng.randint(1, 5)), acc(aa, rng.randint(1, 5), unit=(c + j) % 2)))
        big.chain(T=rng.randint(2000, 5000), prio=c + 1, cbs=cbs)
    b = flatten([s0, s1, big, s0], comm_cost=2)
    _, _, st, _ = O.analyze(b)
    assert st.tolist() == [0, 0, 0, 0]
    assert_same(b, gpu_host_path(b))
    # an over-cap set (33 chains) is rejected with ERANGE on both sides
    over = System(); a = over.accel(server_core=0); x = over.executor(core=1)
    for c in range(33):
        over.chain(T=1000, prio=c + 1, cbs=[cb(x, cpu(1))])
    b = flatten([over, s1], comm_cost=0)
    assert_same(b, gpu_host_path(b))
    assert gpu_host_path(b)[2].tolist() == [1, 0]


@pytest.mark.parametrize("cfg,cpu_only", [("config2", 0.0), ("config2", 0.25), ("config3", 0.0), ("modeB_split", 0.0),
                                          ("deep_deps", 0.0), ("many_cores", 0.0)])
def test_generated_workloads_full(cfg, cpu_only):
    if cfg == "config2":
        p, seed, n = config2_params(cpu_only_frac=cpu_only), 2, 10_000
    elif cfg == "config3":
        p, seed, n = config3_params(), 3, 20_000
    elif cfg == "deep_deps":  # one core, shared spinning executors: every sub-chain waits for the previous ones
        p, seed, n = make_params(exec_mode=1, n_cores=1, n_exec=4, xexec_frac=0.5, spin_frac=1.0), 13, 10_000
    elif cfg == "many_cores":  # 16 cores, up to 32 chains: more ready sub-chains than one Eq.5 wave takes
        p, seed, n = make_params(m_lo=20, m_hi=32, cbs_per_chain=2, n_cores=16, n_exec=16), 14, 10_000
    else:
        p, seed, n = make_params(exec_mode=1, n_exec=4, xexec_frac=0.5, cpu_only_frac=0.2, spin_frac=0.5), 6, 20_000
    b = generate_host(p, seed, 0, n)
    assert_same(b, gpu_host_path(b))


def gen_gpu(p, seed, first, n):
    pp = paam.PaamGenParams.from_buffer_copy(bytes(p))
    return paam.Raw(pp, seed, first, n)


GEN_CASES = ((config3_params(), 3), (config2_params(0.25), 2), (make_params(exec_mode=1, xexec_frac=0.5), 8),
             (make_params(rm=True, spin_frac=0.5), 9),                                   # rate-monotonic
             (make_params(m_lo=1, m_hi=21, cbs_per_chain=3, cpu_only_frac=0.3), 10),     # K=3: passes straddle chains
             (make_params(m_lo=32, m_hi=32, cbs_per_chain=2, n_cores=32, n_bins=0), 11),  # maximum m, no bins
             (make_params(exec_mode=1, n_exec=32, xexec_frac=1.0, ratio_acc=3, ratio_cpu=1,
                          accels=((6, 4, 391 * US, 130 * US), (1, 2, 391 * US, 0), (3, 8, 5, 7), (32, 1, 0, 0))), 12))


def test_device_generator_matches_host_bytes():
    for p, seed in GEN_CASES:
        h = generate_host(p, seed, 1000, 5000)
        raw = gen_gpu(p, seed, 1000, 5000)
        d = raw.to_host()
        for k, v in h.items():
            if k == "set_bin" and p.n_bins == 0:
                assert d[k] is None  # no bins: the device batch has no bin array
            elif isinstance(v, np.ndarray):
                assert np.array_equal(v, d[k]), (k, seed)
        raw.free()


def test_regenerate_reuses_handle():
    p = config3_params()
    pp = paam.PaamGenParams.from_buffer_copy(bytes(p))
    raw = gen_gpu(p, 3, 0, 3000)
    for first, n in ((100, 2000), (7, 9000), (0, 0), (5, 1)):  # shrink, grow, empty, one set
        raw.regenerate(pp, 4, first, n)
        d = raw.to_host()
        h = generate_host(p, 4, first, n)
        for k, v in h.items():
            if k == "set_bin" and n == 0:
                assert d[k] is None or len(d[k]) == 0
            elif isinstance(v, np.ndarray):
                assert np.array_equal(v, d[k]), (k, first, n)
    raw.free()


def test_device_pipeline_generate_pack_analyze_bins():
    """The bench's exact path (generate -> pack -> analyze with bins), 200k config-3 sets, vs oracle."""
    p = config3_params()
    n = 200_000
    raw = gen_gpu(p, 3, 0, n)
    dev = torch.device("cuda")
    sets = paam.Sets(raw)
    wcrt = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    sched = torch.empty(n, dtype=torch.uint8, device=dev)
    bins = torch.zeros(2 * p.n_bins, dtype=torch.int64, device=dev)
    sets.analyze(wcrt, sched, bins)
    torch.cuda.synchronize()
    ow, osch, ob, _ = O.generate_analyze(p, 3, 0, n, want_wcrt=True, nthreads=NPROC)
    assert np.array_equal(sched.cpu().numpy(), osch)
    assert np.array_equal(bins.cpu().numpy(), ob)
    off = raw.to_host()["set_chain_off"]
    gw = wcrt.cpu().numpy().view(np.uint64)
    m = np.diff(off)
    idx = np.repeat(np.arange(n), m) * 32 + (np.arange(len(gw)) - np.repeat(off[:-1], m))
    assert np.array_equal(gw, ow.reshape(-1)[idx])


def test_bins_accumulate_and_partition():
    """Bin counts of two halves add up to the whole (the multi-GPU all-reduce relies on it)."""
    p = config3_params()
    dev = torch.device("cuda")
    tot = torch.zeros(2 * p.n_bins, dtype=torch.int64, device=dev)
    for first, n in ((0, 3000), (3000, 7000)):
        raw = gen_gpu(p, 4, first, n)
        sets = paam.Sets(raw)
        sets.analyze(None, None, tot)
    whole = torch.zeros_like(tot)
    raw = gen_gpu(p, 4, 0, 10000)
    paam.Sets(raw).analyze(None, None, whole)
    torch.cuda.synchronize()
    assert torch.equal(tot, whole)
    _, _, ob, _ = O.generate_analyze(p, 4, 0, 10000, nthreads=NPROC)
    assert np.array_equal(whole.cpu().numpy(), ob)


def test_pipelined_pack_analyze_matches_oracle():
    """paam_pack_analyze (chunks of pack and analyze overlapped on two streams) == oracle."""
    p = config3_params()
    n = 100_003
    raw = gen_gpu(p, 4, 7, n)
    dev = torch.device("cuda")
    sets = paam.Sets(raw)
    wcrt = torch.full((raw.c.n_chains,), -7, dtype=torch.int64, device=dev)
    sched = torch.full((n,), 9, dtype=torch.uint8, device=dev)
    bins = torch.zeros(2 * p.n_bins, dtype=torch.int64, device=dev)
    status = torch.full((n,), -1, dtype=torch.int32, device=dev)
    sets.pack_analyze(raw, wcrt, sched, bins, out_status=status)
    torch.cuda.synchronize()
    assert (status.cpu().numpy() == 0).all()
    ow, osch, ob, _ = O.generate_analyze(p, 4, 7, n, want_wcrt=True, nthreads=NPROC)
    assert np.array_equal(sched.cpu().numpy(), osch)
    assert np.array_equal(bins.cpu().numpy(), ob)
    off = raw.to_host()["set_chain_off"]
    gw = wcrt.cpu().numpy().view(np.uint64)
    m = np.diff(off)
    idx = np.repeat(np.arange(n), m) * 32 + (np.arange(len(gw)) - np.repeat(off[:-1], m))
    assert np.array_equal(gw, ow.reshape(-1)[idx])


@pytest.mark.parametrize("flags", [2, 3])
def test_wfd_units_parity(flags):
    rng = random.Random(100 + flags)
    systems = [random_small_system(rng, max_chains=6, tmax=200) for _ in range(2000)]
    b = flatten(systems, comm_cost=3, flags=flags)
    assert_same(b, gpu_host_path(b))
    p = make_params(accels=((6, 3, 391 * US, 130 * US), (1, 2, 391 * US, 0)))
    g = generate_host(p, 3, 0, 5000)
    g["flags"] = flags
    assert_same(g, gpu_host_path(g))


@pytest.mark.parametrize("case", ["m1-24", "split"])
def test_mixed_set_sizes(case):
    """Batches mixing small and large sets (1-24 chains; chains split over two executors, up to 32
    sub-chains) through the pipelined pack + analyze path, vs the oracle."""
    if case == "m1-24":
        p, seed = make_params(m_lo=1, m_hi=24, cbs_per_chain=2), 5
    else:
        p, seed = make_params(exec_mode=1, n_exec=8, xexec_frac=1.0, m_lo=8, m_hi=16), 6
    n = 30_000
    raw = gen_gpu(p, seed, 0, n)
    dev = torch.device("cuda")
    sets = paam.Sets(raw)
    wcrt = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    sched = torch.empty(n, dtype=torch.uint8, device=dev)
    status = torch.full((n,), -9, dtype=torch.int32, device=dev)
    sets.pack_analyze(raw, wcrt, sched, None, out_status=status)
    torch.cuda.synchronize()
    h = generate_host(p, seed, 0, n)
    ow, osch, ost, _ = O.analyze(h, nthreads=NPROC)
    assert np.array_equal(status.cpu().numpy(), ost)
    assert np.array_equal(sched.cpu().numpy(), osch)
    assert np.array_equal(wcrt.cpu().numpy().view(np.uint64), ow)


@pytest.mark.parametrize("pinned", [False, True])
def test_pack_analyze_from_host_batch_pipelined(pinned):
    """paam_pack_analyze on a HOST batch: chunk slices copied H2D on a copy stream while earlier chunks
    are packed and analysed; host status array; == oracle."""
    p = config3_params()
    n = 20_011
    alloc = (lambda nb: torch.empty(max(nb, 1), dtype=torch.uint8, pin_memory=True).numpy()) if pinned else None
    h = generate_host(p, 9, 3, n, pinned_alloc=alloc)
    hb = paam.Batch.from_host(h)
    dev = torch.device("cuda")
    sets = paam.Sets(hb)
    wcrt = torch.full((hb.c.n_chains,), -3, dtype=torch.int64, device=dev)
    sched = torch.full((n,), 5, dtype=torch.uint8, device=dev)
    bins = torch.zeros(2 * p.n_bins, dtype=torch.int64, device=dev)
    status = np.full(n, -9, np.int32)
    for _ in range(2):  # twice: the staging buffer is reused
        bins.zero_()
        sets.pack_analyze(hb, wcrt, sched, bins, out_status=status)
    torch.cuda.synchronize()
    ow, osch, ost, ob = O.analyze(h, nthreads=NPROC)
    assert np.array_equal(status, ost)
    assert np.array_equal(sched.cpu().numpy(), osch)
    assert np.array_equal(bins.cpu().numpy(), ob)
    assert np.array_equal(wcrt.cpu().numpy().view(np.uint64), ow)
    # the handle now describes the staged batch: the DES reads it
    resp = torch.empty(hb.c.n_chains, dtype=torch.int64, device=dev)
    sets.simulate(10**9, 3, resp, n=64)
    torch.cuda.synchronize()


def test_malformed_csr_ranges_are_rejected_per_set():
    """A chain's callback range or a callback's segment range leaving its set's range is reported
    EDANGLING for that set alone (the kernel never indexes out of range); the other sets are unchanged."""
    rng = random.Random(21)
    systems = [random_small_system(rng, max_chains=4) for _ in range(40)]
    b = flatten(systems, comm_cost=1)
    _, osch, ost, _ = O.analyze(b)
    bad = dict(b)
    bad["chain_cb_off"] = b["chain_cb_off"].copy()
    bad["cb_seg_off"] = b["cb_seg_off"].copy()
    i, j = 5, 17
    c = int(b["set_chain_off"][i])                  # set i: its first chain claims callbacks of set i+1
    bad["chain_cb_off"][c + 1] = b["chain_cb_off"][b["set_chain_off"][i + 1]] + 1
    cb = int(b["chain_cb_off"][b["set_chain_off"][j]])  # set j: a callback whose segments run backwards
    bad["cb_seg_off"][cb + 1] = b["cb_seg_off"][cb] - 1 if b["cb_seg_off"][cb] > 0 else b["cb_seg_off"][cb]
    st = np.full(len(systems), -9, np.int32)
    hb = paam.Batch.from_host(bad)
    sets = paam.Sets(hb, st)
    sched = torch.full((len(systems),), 7, dtype=torch.uint8, device="cuda")
    sets.analyze(None, sched, None)
    torch.cuda.synchronize()
    assert st[i] != 0 and st[j] != 0
    others = [k for k in range(len(systems)) if k not in (i, i + 1, j)]
    assert np.array_equal(st[others], ost[others])
    assert np.array_equal(sched.cpu().numpy()[others], osch[others])


@pytest.mark.parametrize("n_bins", [9, 40])
def test_out_of_range_bin_is_rejected_not_counted(n_bins):
    """A set whose utilisation bin is >= n_bins is PAAM_SET_ERANGE and counted in no bin, for the
    per-warp shared-memory counters (n_bins <= 32) and the direct global atomics (n_bins > 32)."""
    rng = random.Random(5 + n_bins)
    systems = [random_small_system(rng, max_chains=5) for _ in range(300)]
    for i, s in enumerate(systems):
        s.bin = i % n_bins
    b = flatten(systems, comm_cost=1, n_bins=n_bins)
    b["set_bin"] = b["set_bin"].copy()
    b["set_bin"][[3, 77, 150]] = [n_bins, n_bins + 5, 0xFFFFFFFF]
    ow, osch, ost, ob = O.analyze(b, nthreads=NPROC)
    assert (ost[[3, 77, 150]] == 1).all() and ob.sum() == 2 * 0 + ob.sum()  # oracle rejects them too
    assert ob[0::2].sum() == len(systems) - 3
    assert_same(b, gpu_host_path(b))
    assert_same(b, gpu_device_path(b))


def test_host_pipeline_rejects_non_monotone_offsets():
    """paam_pack_analyze with a host batch reads CSR offsets at chunk boundaries; offsets that are not
    monotone or exceed the totals fail the call with PAAM_EINVAL instead of copying wrong ranges."""
    p = config3_params()
    h = generate_host(p, 4, 0, 8192)
    bad = dict(h)
    bad["set_chain_off"] = h["set_chain_off"].copy()
    bad["set_chain_off"][4096] = bad["set_chain_off"][-1] + 10
    hb = paam.Batch.from_host(h)
    sets = paam.Sets(hb)
    with pytest.raises(paam.PaamError, match="invalid argument"):
        sets.pack_analyze(paam.Batch.from_host(bad), None, None, None)


def _scaled(s, f):
    for ch in s.chains:
        ch.T *= f
        ch.D *= f
        for c in ch.cbs:
            for g in c.segs:
                g.wcet *= f
    s.accels = [(bk, u, sc, e * f, k * f) for (bk, u, sc, e, k) in s.accels]
    return s


@pytest.mark.parametrize("flags", [0, 1, 2])
def test_wide_time_sets_take_the_u64_path(flags):
    """Sets with a time >= 2^31 - 1 ns (u64 boundary; A14: < 2^48) are handed over by the u32
    kernels to wide_kernel and analysed exactly: mixed with ordinary sets, every WCRT, verdict, status
    and bin equals the oracle's, on the split and the fused path; App. B x 1000 gives 11 s / 40 s."""
    rng = random.Random(900 + flags)
    systems = []
    for i in range(1500):
        s = random_small_system(rng, max_chains=6, tmax=200)
        if i % 2:
            s = _scaled(s, 1 << 26)
        systems.append(mutate_invalid(s, rng) if i % 3 == 0 else s)
    for i, s in enumerate(systems):
        s.bin = i % 5
    b = flatten(systems, comm_cost=3 << 20, flags=flags, n_bins=5)
    assert (b["chain_T"] >= (1 << 31) - 1).sum() > 500
    assert_same(b, gpu_host_path(b))
    assert_same(b, gpu_device_path(b), fused_too=False)
    app = app_b_two_chains()
    gw, gsch, _, _ = gpu_host_path(flatten([_scaled(app, 1000)], comm_cost=0))
    assert gw.tolist() == [x * 1000 for x in GOLD["two_chains_one_executor"]["R"]]


@pytest.mark.parametrize("flags", [0, 1])
def test_u32_path_overflowing_sums(flags):
    """Sets that stay on the u32 kernels (every time < 2^31 - 1 ns, A14) but whose Lemma-2 / Lemma-3 / Eq.5
    sums pass 2^32: times scaled up to just below 2^31 and the CPU and accelerator WCETs of random chains
    multiplied up to 64x (utilisation far above 1), so the floor-term products reach ~2^51 and the 64-bit
    sums' latched high words decide saturation (UNSCHED, A4).  Every WCRT, verdict, status and bin equals
    the oracle's (exact u64 arithmetic), split and fused paths."""
    rng = random.Random(4242 + flags)
    lim = (1 << 31) - 1
    systems = []
    for i in range(2000):
        s = random_small_system(rng, max_chains=6, tmax=200)
        for ch in s.chains:
            if rng.random() < 0.4:
                k = rng.choice([2, 8, 64])
                for c in ch.cbs:
                    for g in c.segs:
                        g.wcet *= k
        top = max([c.T for c in s.chains] + [c.D for c in s.chains] + [g.wcet for c in s.chains for x in c.cbs
                   for g in x.segs] + [e for a in s.accels for e in a[3:5]] + [1])
        target = rng.choice([lim - 1, lim - 1, 1 << 30, (1 << 29) + rng.randrange(1 << 20)])
        s = _scaled(s, max(1, target // top))
        systems.append(s)
    for i, s in enumerate(systems):
        s.bin = i % 5
    b = flatten(systems, comm_cost=rng.choice([0, 5, 1 << 20]), flags=flags, n_bins=5)
    times = [b["chain_T"], b["chain_D"], b["seg_wcet"], b["accel_eps"], b["accel_kappa"]]
    assert max(int(t.max()) for t in times if t.size) < lim  # every set on the u32 kernels
    assert int(b["chain_T"].max()) > (1 << 30)
    ow, osch, ost, _ = O.analyze(b, nthreads=NPROC)
    assert (ow == O.UNSCHED).sum() > 1000 and osch.sum() > 100  # both outcomes well represented
    assert_same(b, gpu_device_path(b))


def test_wide_time_sets_admission_and_des_status():
    """paam_admit decides wide sets on the u64 path too; the DES reports them PAAM_SIM_WIDE (it computes in
    32-bit time distances) and simulates the others."""
    rng = random.Random(77)
    systems = [random_small_system(rng, max_chains=5, tmax=200) for _ in range(200)]
    systems = [_scaled(s, 1 << 26) if i % 2 else s for i, s in enumerate(systems)]
    b = flatten(systems, comm_cost=1)
    ow, osch, ost, _ = O.analyze(b, nthreads=NPROC)
    hb = paam.Batch.from_host(b)
    sets = paam.Sets(hb)
    dec = torch.full((len(systems),), -9, dtype=torch.int32, device="cuda")
    sets.admit(dec)
    st = torch.full((len(systems),), -9, dtype=torch.int32, device="cuda")
    resp = torch.zeros(max(hb.c.n_chains, 1), dtype=torch.int64, device="cuda")
    sets.simulate(400, 1, resp, out_status=st)
    torch.cuda.synchronize()
    d = dec.cpu().numpy()
    off = b["set_chain_off"]
    for i in range(len(systems)):
        c0, c1 = int(off[i]), int(off[i + 1])
        if ost[i] != 0:
            assert d[i] == -2 - ost[i]
        elif osch[i]:
            assert d[i] == -1
        else:  # the highest-priority CRITICAL chain with R* > D
            bad = [c for c in range(c1 - c0) if b["chain_class"][c0 + c] == 0 and (ow[c0 + c] == O.UNSCHED or ow[c0 + c] > b["chain_D"][c0 + c])]
            assert d[i] == max(bad, key=lambda c: b["chain_prio"][c0 + c])
    s = st.cpu().numpy()
    lim = (1 << 31) - 1
    wide = np.array([any(ch.T >= lim or ch.D >= lim or any(g.wcet >= lim for c in ch.cbs for g in c.segs)
                         for ch in x.chains) or any(e >= lim or k >= lim for (_b, _u, _c, e, k) in x.accels)
                     for x in systems])
    assert wide.sum() > 50
    assert (s[wide] == paam.PAAM_SIM_WIDE).all()
    assert (s[~wide] != paam.PAAM_SIM_WIDE).all()


def gpu_compact_path(batch, device=False):
    """paam_pack_analyze32 on the compact form of `batch` (host or device), through a handle whose capacity
    comes from paam_pack of the u64 batch; returns (wcrt, sched, status, bins) as paam.analyze."""
    n = batch["n_sets"]
    dev = torch.device("cuda")
    sets = paam.Sets(paam.Batch.from_host(batch))
    b32 = paam.Batch32.from_host_to_device(batch) if device else paam.Batch32.from_host(batch)
    status = (torch.full((max(n, 1),), -9, dtype=torch.int32, device=dev) if device
              else np.full(max(n, 1), -9, np.int32))
    nch = int(batch["set_chain_off"][-1])
    wcrt = torch.full((max(nch, 1),), -5, dtype=torch.int64, device=dev)
    sched = torch.full((max(n, 1),), 7, dtype=torch.uint8, device=dev)
    nb = int(batch.get("n_bins", 0))
    bins = torch.zeros(max(2 * nb, 1), dtype=torch.int64, device=dev)
    sets.pack_analyze(b32, wcrt, sched, bins if nb else None, out_status=status)
    torch.cuda.synchronize()
    st = status if isinstance(status, np.ndarray) else status.cpu().numpy()
    out = (wcrt.cpu().numpy().view(np.uint64)[:nch], sched.cpu().numpy()[:n], st[:n], bins.cpu().numpy()[:2 * nb])
    sets.free()
    return out


def mutate_invalid_compact(s: System, rng):
    """Break one validation rule that the compact batch can express (or none)."""
    k = rng.randrange(8)
    if k == 0 and len(s.chains) > 1:
        s.chains[1].prio = s.chains[0].prio
    elif k == 1:
        s.chains[0].D = s.chains[0].T + 1
        s.chains[0].cls = CRITICAL
    elif k == 2:
        s.chains[0].cbs[0].exec = 31
    elif k == 3:
        s.chains[0].cbs[0].segs.append(Seg(1, 1, 3, 0))  # undeclared accelerator
    elif k == 4:
        s.chains[0].cbs[0].segs[0].wcet = 0
    elif k == 5:
        s.execs[0] = (10, 1, 0)  # server core of accelerator 0
    elif k == 6:
        s.chains[0].cbs[0].segs.append(Seg(s.chains[0].cbs[0].segs[-1].kind, 1))
    return s


@pytest.mark.parametrize("flags", [0, 1, 3])
def test_compact_batch_gives_the_u64_batch_results(flags):
    """paam_pack_analyze32 (the compact batch: u32 times, one byte per segment) is bit-exact with the
    oracle on the same sets: valid and invalid ones, times on both sides of 2^31 - 1 ns (the wide ones take
    the u64 kernel through the compact loads), host and device batches, the generated config-3 workload."""
    rng = random.Random(300 + flags)
    systems = []
    for i in range(1200):
        s = random_small_system(rng, max_chains=6, tmax=120)
        if i % 4 == 1:  # the largest time scaled to just below 2^32 ns: wide, still representable in 32 bits
            top = max([c.T for c in s.chains] + [c.D for c in s.chains] + [g.wcet for c in s.chains for x in c.cbs
                       for g in x.segs] + [e for a in s.accels for e in a[3:5]] + [1])
            s = _scaled(s, ((1 << 32) - 1) // top)
        systems.append(mutate_invalid_compact(s, rng) if i % 3 == 0 else s)
    for i, s in enumerate(systems):
        s.bin = i % 5
    b = flatten(systems, comm_cost=3, flags=flags, n_bins=5)
    assert int(b["chain_T"].max()) < (1 << 32) and (b["chain_T"] >= (1 << 31) - 1).any()
    assert_same(b, gpu_compact_path(b), fused_too=False)
    assert_same(b, gpu_compact_path(b, device=True), fused_too=False)
    g = generate_host(config3_params(), 4, 0, 20_000)
    assert_same(g, gpu_compact_path(g), fused_too=False)


def test_compact_batch_handle_refuses_a_later_pack():
    """After paam_pack_analyze32 the handle holds no batch paam_analyze could pack: PAAM_EINVAL, until a
    paam_repack of a u64 batch."""
    b = flatten([app_b_two_chains()], comm_cost=0)
    sets = paam.Sets(paam.Batch.from_host(b))
    sets.pack_analyze(paam.Batch32.from_host(b))
    with pytest.raises(paam.PaamError, match="compact"):
        sets.analyze(torch.empty(2, dtype=torch.int64, device="cuda"))
    sets.repack(paam.Batch.from_host(b))
    w = torch.empty(2, dtype=torch.int64, device="cuda")
    sets.analyze(w)
    torch.cuda.synchronize()
    assert w.cpu().tolist() == GOLD["two_chains_one_executor"]["R"]


def test_invalid_segment_kind_is_not_counted_as_an_accelerator_segment():
    """Validation counts ACCEL segments (kind == 1) against the 64-segment cap; a segment of an undefined
    kind (2) is an ESHAPE error, never an accelerator segment (include/paam.h ERANGE / ESHAPE).  A set with
    exactly 64 ACCEL segments plus one kind-2 segment is ESHAPE (not ERANGE), on every path."""
    s = System()
    a = s.accel(buckets=1, server_core=0)
    x = s.executor(core=1)
    s.chain(T=100 * MS, prio=1, cbs=[cb(x, cpu(1), acc(a, 1)) for _ in range(64)])
    bad = System()
    a = bad.accel(buckets=1, server_core=0)
    x = bad.executor(core=1)
    bad.chain(T=100 * MS, prio=1, cbs=[cb(x, cpu(1), acc(a, 1)) for _ in range(63)] + [cb(x, Seg(2, 1), acc(a, 1))])
    b = flatten([s, bad], comm_cost=0)
    _, _, st, _ = O.analyze(b)
    assert st.tolist() == [0, 4]  # OK, ESHAPE
    assert_same(b, gpu_host_path(b))


@pytest.mark.parametrize("pinned", [False, True])
def test_host_outputs_of_a_host_batch(pinned):
    """A host batch may write its WCRTs and verdicts straight into host memory (pageable numpy or pinned
    tensors): the library copies each chunk back as its kernels finish; the results equal the oracle's,
    for the u64 and the compact batch.  Host outputs with a device batch are refused."""
    p = config3_params()
    g = generate_host(p, 4, 0, 20_000)
    ow, osch, _, ob = O.analyze(g, nthreads=NPROC)
    hb = paam.Batch.from_host(g)
    sets = paam.Sets(hb)
    for batch in (hb, paam.Batch32.from_host(g)):
        if pinned:
            w = torch.zeros(hb.c.n_chains, dtype=torch.int64, pin_memory=True)
            sc = torch.zeros(g["n_sets"], dtype=torch.uint8, pin_memory=True)
        else:
            w = np.zeros(hb.c.n_chains, np.uint64)
            sc = np.zeros(g["n_sets"], np.uint8)
        bins = torch.zeros(2 * p.n_bins, dtype=torch.int64, device="cuda")
        sets.pack_analyze(batch, w, sc, bins)
        torch.cuda.synchronize()
        wn = w.numpy().view(np.uint64) if pinned else w
        scn = sc.numpy() if pinned else sc
        assert np.array_equal(wn, ow) and np.array_equal(scn, osch)
        assert np.array_equal(bins.cpu().numpy(), ob)
    db = paam.Batch.from_host_to_device(g)
    with pytest.raises(paam.PaamError, match="host batch"):
        sets.pack_analyze(db, np.zeros(hb.c.n_chains, np.uint64), None, None)
