"""Batched admission what-if (paam_admit) vs the oracle."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen.inputs import CRITICAL, MS, System, acc, cb, cpu, flatten, with_candidate
from oracle import oracle as O
from paper_2404_06452_b200 import paam
from tests.ref_scan import random_small_system
from tests.test_oracle_pins import cs3_system


def gpu_admit(systems):
    hb = paam.Batch.from_host(flatten(systems, comm_cost=1))
    sets = paam.Sets(hb)
    dec = torch.empty(max(hb.n_sets, 1), dtype=torch.int32, device="cuda")
    sets.admit(dec)
    torch.cuda.synchronize()
    return dec.cpu().numpy()[:hb.n_sets]


def oracle_decision(systems):
    b = flatten(systems, comm_cost=1)
    w, _, st, _ = O.analyze(b)
    off = b["set_chain_off"]
    out = []
    for i, s in enumerate(systems):
        if st[i] != 0:
            out.append(-2 - int(st[i]))
            continue
        fails = [(s.chains[c].prio, c) for c in range(len(s.chains))
                 if s.chains[c].cls == CRITICAL and (w[off[i] + c] == O.UNSCHED or w[off[i] + c] > s.chains[c].D)]
        out.append(max(fails)[1] if fails else -1)
    return np.array(out, np.int32)


def test_spec_examples():
    base = cs3_system(6)  # schedulable (Case Study 3)
    x = base.executor(core=7)
    g = 0
    # a vanishing candidate (1 ns of CPU, huge period, lowest priority, own core) is accepted;
    # one that also used the GPU would change the bucket map (7 users of 6 buckets) and break chain 2
    tiny = with_candidate(base, T=2000 * MS, prio=0, cbs=[cb(x, cpu(1))])
    hog = with_candidate(base, T=100 * MS, prio=100, cbs=[cb(x, cpu(1 * MS), acc(g, 10 * MS))])
    selfish = with_candidate(base, T=10 * MS, D=10 * MS, prio=8, cbs=[cb(x, cpu(20 * MS))])   # S:244 REJECT(itself)
    dup = with_candidate(base, T=1000 * MS, prio=6, cbs=[cb(x, cpu(1))])                     # duplicate priority
    systems = [tiny, hog, selfish, dup]
    got = gpu_admit(systems)
    assert got.tolist() == oracle_decision(systems).tolist()
    assert got[0] == -1
    assert got[1] == 1  # the new highest-priority chain breaks existing chain 2 (index 1)
    assert got[2] == len(selfish.chains) - 1
    assert got[3] == -2 - 5  # PAAM_SET_EDUPPRIO


def test_random_what_if_matches_oracle():
    rng = random.Random(8)
    systems = []
    for _ in range(2000):
        s = random_small_system(rng, max_chains=5, tmax=100)
        x = rng.randrange(len(s.execs))
        prio = rng.choice([ch.prio for ch in s.chains] + [50, 60])  # sometimes a duplicate
        systems.append(with_candidate(s, T=rng.randint(20, 100), prio=prio,
                                      cbs=[cb(x, cpu(rng.randint(1, 4)), acc(0, rng.randint(1, 6)))]))
    got = gpu_admit(systems)
    assert np.array_equal(got, oracle_decision(systems))
    assert (got == -1).any() and (got >= 0).any() and (got <= -2).any()
