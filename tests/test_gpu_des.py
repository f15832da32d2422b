"""GPU parity of paam_simulate (DES kernel) with the oracle DES: per-chain maximum response, completed
instance counts, per-set event digests and sim <= bound violation counts, bit-exact."""
import os
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen.inputs import MS, config2_params, config3_params, flatten, generate_host, make_params
from oracle import oracle as O
from paper_2404_06452_b200 import paam
from tests.ref_scan import random_small_system
from tests.test_oracle_pins import a10_system, app_b_two_chains, cs3_system, two_chain_accel_system

NPROC = os.cpu_count() or 1


def gpu_sim(batch, horizon, seed, first_index=0, with_bound=True):
    dev = torch.device("cuda")
    hb = paam.Batch.from_host(batch)
    sets = paam.Sets(hb)
    nch = max(hb.c.n_chains, 1)
    bound = None
    if with_bound:
        bound = torch.empty(nch, dtype=torch.int64, device=dev)
        sets.analyze(bound, None, None)
    resp = torch.zeros(nch, dtype=torch.int64, device=dev)
    cnt = torch.zeros(nch, dtype=torch.int64, device=dev)
    dig = torch.zeros(max(hb.n_sets, 1), dtype=torch.int64, device=dev)
    viol = torch.zeros(1, dtype=torch.int64, device=dev)
    sets.simulate(horizon, seed, resp, cnt, dig, bound, viol, first_index=first_index)
    torch.cuda.synchronize()
    out = dict(resp=resp.cpu().numpy().view(np.uint64)[:hb.c.n_chains], count=cnt.cpu().numpy().view(np.uint64)[:hb.c.n_chains],
               digest=dig.cpu().numpy().view(np.uint64)[:hb.n_sets], violations=int(viol.item()),
               bound=None if bound is None else bound.cpu().numpy().view(np.uint64)[:hb.c.n_chains])
    sets.free()
    return out


def check(batch, horizon, seed, first_index=0):
    g = gpu_sim(batch, horizon, seed, first_index)
    o = O.simulate(batch, horizon, seed=seed, first_index=first_index, bound=g["bound"], nthreads=NPROC)
    bad = np.nonzero(o["resp"] != g["resp"])[0]
    assert bad.size == 0, (bad[:5], o["resp"][bad[:5]], g["resp"][bad[:5]])
    assert np.array_equal(o["count"], g["count"])
    badd = np.nonzero(o["digest"] != g["digest"])[0]
    assert badd.size == 0, badd[:10]
    assert o["violations"] == g["violations"]
    return o


def test_worked_examples_des():
    systems = [two_chain_accel_system(kappa=100_000, buckets=2), app_b_two_chains(), cs3_system(6), cs3_system(1),
               a10_system()]
    b = flatten(systems, comm_cost=0)
    for seed in (0, 1, 2, 3):
        check(b, 1_500 * MS, seed)


@pytest.mark.parametrize("seed", [0, 5, 9])
def test_random_small_systems_des(seed):
    rng = random.Random(400 + seed)
    systems = [random_small_system(rng, max_chains=6, tmax=60) for _ in range(600)]
    b = flatten(systems, comm_cost=2)
    _, _, st, _ = O.analyze(b)
    assert (st == 0).all()
    check(b, 400, seed)


def test_random_small_systems_des_zero_comm():
    """comm = 0 with eps / kappa often 0: zero-length transits, eps phases and switches, so settle
    passes repeat at one timestamp (the pass-repeat rules of simulate.cu)."""
    rng = random.Random(977)
    systems = [random_small_system(rng, max_chains=6, tmax=60) for _ in range(600)]
    b = flatten(systems, comm_cost=0)
    _, _, st, _ = O.analyze(b)
    assert (st == 0).all()
    check(b, 400, 4)


@pytest.mark.parametrize("cfg", ["config3", "config2_cpuonly", "modeB_split"])
def test_generated_des(cfg):
    if cfg == "config3":
        p, seed, n = config3_params(), 3, 400
    elif cfg == "config2_cpuonly":
        p, seed, n = config2_params(cpu_only_frac=0.25), 2, 400
    else:
        p, seed, n = make_params(exec_mode=1, n_exec=4, xexec_frac=0.5, spin_frac=0.5, cpu_only_frac=0.2), 6, 400
    b = generate_host(p, seed, 1000, n)
    o = check(b, 10_000 * MS, seed=11, first_index=1000)
    assert o["count"].sum() > 100 * n


def test_des_first_index_shards_compose():
    """Digests depend on (seed, global set index) only: two shards equal the whole (G-invariance)."""
    p = config3_params()
    whole = generate_host(p, 5, 0, 64)
    g = gpu_sim(whole, 3_000 * MS, 7, first_index=0, with_bound=False)
    a = gpu_sim(generate_host(p, 5, 0, 32), 3_000 * MS, 7, first_index=0, with_bound=False)
    b2 = gpu_sim(generate_host(p, 5, 32, 32), 3_000 * MS, 7, first_index=32, with_bound=False)
    assert np.array_equal(np.concatenate([a["digest"], b2["digest"]]), g["digest"])


def gpu_sim_fifo(batch, horizon, seed):
    dev = torch.device("cuda")
    hb = paam.Batch.from_host(batch)
    sets = paam.Sets(hb)
    nch = max(hb.c.n_chains, 1)
    resp = torch.zeros(nch, dtype=torch.int64, device=dev)
    cnt = torch.zeros(nch, dtype=torch.int64, device=dev)
    dig = torch.zeros(max(hb.n_sets, 1), dtype=torch.int64, device=dev)
    sets.simulate(horizon, seed, resp, cnt, dig, fifo=True)
    torch.cuda.synchronize()
    return (resp.cpu().numpy().view(np.uint64)[:hb.c.n_chains], cnt.cpu().numpy().view(np.uint64)[:hb.c.n_chains],
            dig.cpu().numpy().view(np.uint64)[:hb.n_sets])


def test_fifo_direct_parity_and_comparison():
    rng = random.Random(31)
    systems = [random_small_system(rng, max_chains=6, tmax=60) for _ in range(400)] + [cs3_system(6), cs3_system(1)]
    b = flatten(systems, comm_cost=1)
    for seed in (0, 4):
        g = gpu_sim_fifo(b, 500, seed)
        o = O.simulate(b, 500, seed=seed, nthreads=NPROC, fifo=True)
        assert np.array_equal(g[0], o["resp"]) and np.array_equal(g[1], o["count"]) and np.array_equal(g[2], o["digest"])
    cs = flatten([cs3_system(6)], comm_cost=0)
    paam_r = gpu_sim(cs, 3_000 * MS, 1)
    fifo_r = gpu_sim_fifo(cs, 3_000 * MS, 1)
    assert paam_r["resp"][0] <= paam_r["bound"][0] and paam_r["resp"][0] <= 0.8 * fifo_r[0][0]


def test_des_wfd_units_parity():
    rng = random.Random(55)
    systems = [random_small_system(rng, max_chains=6, tmax=60) for _ in range(300)]
    b = flatten(systems, comm_cost=1, flags=2)
    check(b, 400, 3)
