"""Oracle pins: worked examples with fixed expected values (tests/golden/worked_examples.json).

Every expected value below comes from the paper / SPEC worked examples or from a hand derivation
cited in the golden file -- never from the code under test.
"""
import ctypes
import json
import os

import numpy as np
import pytest

from gen.inputs import (BEST_EFFORT, CRITICAL, MS, SPIN, SUSPEND, US, System, acc, cb, cpu, flatten)
from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
UNSCHED = O.UNSCHED


def unsched(v):
    return UNSCHED if v == "UNSCHED" else v


def run(systems, comm=0, flags=0):
    b = flatten(systems, comm_cost=comm, flags=flags)
    return b, O.analyze(b)


def test_mu_examples():
    O.lib().oracle_mu.restype = ctypes.c_uint64
    O.lib().oracle_mu.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    for t, T, want in GOLD["mu"]["cases"]:
        assert O.lib().oracle_mu(t, T) == want


def test_lemma2_lone_segment():
    s = System()
    a = s.accel(buckets=1, server_core=0)
    x = s.executor(core=1)
    s.chain(T=20 * MS, prio=1, cbs=[cb(x, acc(a, 3 * MS))])
    b, _ = run([s])
    assert O.detail(b)["aseg_H"] == [GOLD["lemma2_lone"]["H"]]


def two_chain_accel_system(kappa=0, eps=0, buckets=1):
    """HP chain (A=3ms, T=20ms) and LP chain (A=5ms, T=50ms) on one accelerator, own executors."""
    s = System()
    a = s.accel(buckets=buckets, server_core=0, eps=eps, kappa=kappa)
    x1 = s.executor(core=1)
    x2 = s.executor(core=2)
    s.chain(T=20 * MS, prio=2, cbs=[cb(x1, acc(a, 3 * MS))])
    s.chain(T=50 * MS, prio=1, cbs=[cb(x2, acc(a, 5 * MS))])
    return s


def test_lemma2_blocker_and_interference():
    b, _ = run([two_chain_accel_system()])
    d = O.detail(b)
    assert d["aseg_LPB"] == [5 * MS, 0]
    assert d["aseg_H"][0] == GOLD["lemma2_hp_vs_lp_blocker"]["H"]
    assert d["aseg_H"][1] == GOLD["lemma2_lp_vs_hp"]["H"]


def test_lemma3_at_R25():
    # LP chain: CPU 14ms + own A=5ms; HP interferer A=3ms T=20ms elsewhere.  F(R) = 14 + min(11, C(R)),
    # so R converges to 25ms where C(25) = 5 + (ceil(25/20)+1)*3 = 14.
    s = System()
    a = s.accel(buckets=1, server_core=0)
    x1 = s.executor(core=1)
    x2 = s.executor(core=2)
    s.chain(T=20 * MS, prio=2, cbs=[cb(x1, acc(a, 3 * MS))])
    s.chain(T=100 * MS, prio=1, cbs=[cb(x2, cpu(14 * MS), acc(a, 5 * MS))])
    b, _ = run([s])
    d = O.detail(b)
    g = GOLD["lemma3_at_25"]
    assert d["sub_R"][1] == g["R"]
    assert d["sub_C"][1] == g["C"]
    assert d["sub_Hstar"][1] == g["Hstar"]


def test_eq1_overhead():
    b, _ = run([two_chain_accel_system(eps=391 * US)])
    d = O.detail(b)
    assert d["sub_Hstar"][0] == GOLD["eq1"]["Hstar"]


def test_blocking_examples():
    want = GOLD["blocking"]["B"]
    # (a) no LP chain on the executor
    s = System(); s.accel(server_core=0); x = s.executor(core=1)
    s.chain(T=100 * MS, prio=1, cbs=[cb(x, cpu(1 * MS))])
    assert O.detail(flatten([s]))["sub_B"] == [want[0]]
    # (b) one LP chain with callbacks E = {4, 7}
    s = System(); s.accel(server_core=0); x = s.executor(core=1)
    s.chain(T=100 * MS, prio=2, cbs=[cb(x, cpu(1 * MS))])
    s.chain(T=100 * MS, prio=1, cbs=[cb(x, cpu(4 * MS)), cb(x, cpu(7 * MS))])
    assert O.detail(flatten([s]))["sub_B"][0] == want[1]
    # (c) two LP chains with maxima 7 and 9
    s = System(); s.accel(server_core=0); x = s.executor(core=1)
    s.chain(T=100 * MS, prio=3, cbs=[cb(x, cpu(1 * MS))])
    s.chain(T=100 * MS, prio=2, cbs=[cb(x, cpu(4 * MS)), cb(x, cpu(7 * MS))])
    s.chain(T=100 * MS, prio=1, cbs=[cb(x, cpu(9 * MS)), cb(x, cpu(2 * MS))])
    assert O.detail(flatten([s]))["sub_B"][0] == want[2]


def test_isolated_chain():
    s = System(); a = s.accel(server_core=0); x = s.executor(core=1)
    s.chain(T=20 * MS, prio=1, cbs=[cb(x, cpu(2 * MS), acc(a, 3 * MS))])
    _, (wcrt, sched, status, _) = run([s])
    assert wcrt.tolist() == [GOLD["isolated"]["R"]] and sched[0] == 1 and status[0] == 0


def test_end_to_end_two_subchains():
    # two sub-chains on two executors (different cores): R = 5 + 7, + 0.1ms comm
    s = System(); s.accel(server_core=0)
    x1 = s.executor(core=1); x2 = s.executor(core=2)
    s.chain(T=100 * MS, prio=1, cbs=[cb(x1, cpu(5 * MS)), cb(x2, cpu(7 * MS))])
    _, (wcrt, sched, _, _) = run([s], comm=100 * US)
    assert wcrt.tolist() == [GOLD["end_to_end"]["R"]]


def app_b_two_chains():
    s = System()
    a = s.accel(buckets=1, server_core=0)
    x = s.executor(core=1)
    s.chain(T=20 * MS, prio=2, cbs=[cb(x, cpu(1 * MS), acc(a, 3 * MS))])
    s.chain(T=50 * MS, prio=1, cbs=[cb(x, cpu(2 * MS), acc(a, 5 * MS))])
    return s


def test_two_chains_one_executor():
    b, (wcrt, sched, _, _) = run([app_b_two_chains()])
    g = GOLD["two_chains_one_executor"]
    assert wcrt.tolist() == g["R"]
    assert sched[0] == 1
    assert O.detail(b)["sub_iters"][1] == len(g["iterates_R2"])


def cs3_system(buckets):
    """Case Study 3: two critical chains T=120/220ms + four BE chains T=52ms, each one
    callback CPU 1ms + GPU 50ms + CPU 1ms, six executors on own cores, server on core 0."""
    s = System()
    g = s.accel(buckets=buckets, units=1, server_core=0, eps=391 * US, kappa=130 * US)
    specs = [(120, 6, CRITICAL), (220, 5, CRITICAL), (52, 4, BEST_EFFORT), (52, 3, BEST_EFFORT),
             (52, 2, BEST_EFFORT), (52, 1, BEST_EFFORT)]
    for i, (T, prio, cls) in enumerate(specs):
        x = s.executor(core=1 + i, prio=1, wait=SUSPEND)
        s.chain(T=T * MS, prio=prio, cls=cls, cbs=[cb(x, cpu(1 * MS), acc(g, 50 * MS), cpu(1 * MS))])
    return s


@pytest.mark.parametrize("buckets,key", [(6, "cs3_n6"), (1, "cs3_n1")])
def test_case_study_3(buckets, key):
    _, (wcrt, sched, status, _) = run([cs3_system(buckets)])
    g = GOLD[key]
    assert status[0] == 0
    assert wcrt[:2].tolist() == [unsched(v) for v in g["R"]]
    assert sched[0] == g["sched"]


def a10_system():
    s = System()
    a = s.accel(buckets=1, server_core=0)
    x = s.executor(core=1)
    s.chain(T=20 * MS, prio=2, cbs=[cb(x, cpu(1 * MS))])
    s.chain(T=50 * MS, prio=1, cbs=[cb(x, cpu(2 * MS), acc(a, 5 * MS))])
    return s


def test_a10_counterexample_as_written_and_sound():
    _, (wcrt, _, _, _) = run([a10_system()])
    assert wcrt.tolist() == GOLD["a10_counterexample"]["R"]
    # sound variant: B_1 = E_j + H + eps of the LP callback = 2 + 5 = 7 -> R1 = 7 + 1 = 8ms
    _, (wcrt, _, _, _) = run([a10_system()], flags=1)
    assert wcrt[0] == 8 * MS


@pytest.mark.parametrize("m,n,want", [
    (6, 6, [5, 4, 3, 2, 1, 0]),
    (12, 6, [5, 5, 4, 4, 3, 3, 2, 2, 1, 1, 0, 0]),
    (5, 1, [0, 0, 0, 0, 0]),
    (7, 6, [5, 5, 4, 4, 3, 3, 2]),                            # A5: groups of ceil(7/6)=2, short group lowest
    (3, 6, [5, 4, 3]),                                        # A5: m < n leaves low buckets empty
])
def test_bucket_map(m, n, want):
    s = System()
    a = s.accel(buckets=n, server_core=0)
    for i in range(m):
        x = s.executor(core=1 + i)
        s.chain(T=1000 * MS, prio=m - i, cbs=[cb(x, acc(a, 1 * MS))])  # chain i has rank i
    d = O.detail(flatten([s]))
    assert d["aseg_bucket"] == want


@pytest.mark.parametrize("mutate,code", [
    (lambda s: s.chains.__setitem__(1, s.chains[1].__class__(s.chains[1].T, s.chains[1].D, 2, 0, s.chains[1].cbs)), 5),
    (lambda s: setattr(s.chains[0], "D", s.chains[0].T + 1), 6),
    (lambda s: setattr(s.chains[0].cbs[0], "exec", 7), 2),
    (lambda s: setattr(s.chains[0].cbs[0].segs[1], "accel", 3), 3),
    (lambda s: setattr(s.chains[0].cbs[0].segs[0], "wcet", 0), 4),
    (lambda s: s.execs.__setitem__(0, (0, 1, 0)), 7),
    (lambda s: setattr(s.chains[0], "T", 1 << 48), 1),
    (lambda s: s.chains[0].cbs[0].segs.append(acc(0, 1)), 4),
])
def test_validation(mutate, code):
    s = app_b_two_chains()
    s.executor(core=2)
    mutate(s)
    _, (wcrt, sched, status, _) = run([s])
    assert status[0] == code
    assert sched[0] == 0 and all(w == UNSCHED for w in wcrt)


def test_validation_noncontiguous_revisit():
    s = System(); s.accel(server_core=0)
    x1 = s.executor(core=1); x2 = s.executor(core=2)
    s.chain(T=100 * MS, prio=1, cbs=[cb(x1, cpu(1)), cb(x2, cpu(1)), cb(x1, cpu(1))])
    _, (_, _, status, _) = run([s])
    assert status[0] == 4


def test_empty_set_is_vacuously_schedulable():
    s = System(); s.accel(server_core=0)
    _, (wcrt, sched, status, _) = run([s])
    assert status[0] == 0 and sched[0] == 1 and wcrt.size == 0


def _wfd_system(utils):
    s = System()
    a = s.accel(buckets=1, units=2, server_core=0)
    for i, A in enumerate(utils):
        x = s.executor(core=1 + i)
        s.chain(T=100, prio=len(utils) - i, cbs=[cb(x, acc(a, A))])
    return s


def test_wfd_unit_assignment():
    """PAAM_FLAG_WFD_UNITS: by decreasing utilisation onto the least-loaded unit.
    [0.4, 0.3, 0.2] -> {0.4} and {0.3, 0.2} (the rule of S:101; the example at S:104 lists
    {0.4, 0.2}/{0.3}, which is not worst fit -- DESIGN.md reading W).  Observed through LP blocking:
    only chains sharing a unit block each other (one bucket)."""
    d = O.detail(flatten([_wfd_system([40, 30, 20])], comm_cost=0, flags=2))
    assert d["aseg_LPB"] == [0, 20, 0]
    # equal utilisations alternate units: u0 {c0, c2}, u1 {c1, c3}
    d = O.detail(flatten([_wfd_system([20, 20, 20, 20])], comm_cost=0, flags=2))
    assert d["aseg_LPB"] == [20, 20, 0, 0]
    # without the flag the input units (all 0) are used: everyone blocks everyone below
    d = O.detail(flatten([_wfd_system([20, 20, 20, 20])], comm_cost=0, flags=0))
    assert d["aseg_LPB"] == [20, 20, 20, 0]


def spin_system(wait):
    """hpp interferer with an accelerator segment (golden 'spin_hpp')."""
    s = System()
    a = s.accel(buckets=1, server_core=0, eps=1 * MS)
    xh = s.executor(core=1, prio=2, wait=wait)
    xc = s.executor(core=1, prio=1, wait=SUSPEND)
    s.chain(T=100 * MS, prio=2, cbs=[cb(xh, cpu(2 * MS), acc(a, 10 * MS))])
    s.chain(T=100 * MS, prio=1, cbs=[cb(xc, cpu(5 * MS))])
    return s


@pytest.mark.parametrize("wait,key", [(SPIN, "R_c_spin"), (SUSPEND, "R_c_suspend")])
def test_spin_of_hpp_interferer(wait, key):
    g = GOLD["spin_hpp"]
    b, (wcrt, sched, status, _) = run([spin_system(wait)])
    d = O.detail(b)
    assert status[0] == 0
    assert d["sub_R"][0] == g["R_h"] and d["sub_Hstar"][0] == g["Hstar_h"]
    assert d["sub_R"][1] == g[key]
    assert wcrt.tolist() == [g["R_h"], g[key]]


def lemma3_union_system():
    """Two segments of one sub-chain on one unit sharing one HP interferer (golden 'lemma3_union')."""
    s = System()
    a = s.accel(buckets=1, server_core=0)
    xh = s.executor(core=2)
    xc = s.executor(core=1)
    s.chain(T=50 * MS, prio=2, cbs=[cb(xh, acc(a, 4 * MS))])
    s.chain(T=200 * MS, prio=1, cbs=[cb(xc, acc(a, 3 * MS), cpu(1 * MS), acc(a, 3 * MS))])
    return s


def test_lemma3_union_counts_each_hp_segment_once():
    g = GOLD["lemma3_union"]
    b, (wcrt, sched, status, _) = run([lemma3_union_system()])
    d = O.detail(b)
    assert status[0] == 0
    assert d["sub_S"][1] == g["S_c"]
    assert d["sub_C"][1] == g["C_c"] and d["sub_Hstar"][1] == g["Hstar_c"]
    assert d["sub_R"][1] == g["R_c"] and wcrt[1] == g["R_c"]
    assert g["R_c"] != g["R_c_if_summed_per_segment"]


def test_out_of_range_bin_is_a_range_error():
    """A utilisation bin outside [0, n_bins) rejects the set (ERANGE, reading V) and counts it nowhere."""
    s = two_chain_accel_system()
    b = flatten([s, s, s], comm_cost=0, n_bins=2)
    b["set_bin"] = np.array([0, 2, 1], np.uint32)
    _, sched, status, bins = O.analyze(b)
    assert status.tolist() == [0, 1, 0] and sched.tolist() == [1, 0, 1]
    assert bins.tolist() == [1, 1, 1, 1]


def test_wide_times_scale_exactly():
    """Times of 2^31 ns and beyond (u64 boundary; domain < 2^48 ns, A14): the analysis is
    homogeneous of degree one in time (mu(R, T) = ceil(R/T) + 1 is scale-invariant), so App. B's
    two-chain set with every time x1000 (T = 20 s / 50 s) has R = 11 s / 40 s exactly."""
    s = app_b_two_chains()
    for ch in s.chains:
        ch.T *= 1000
        ch.D *= 1000
        for c in ch.cbs:
            for g in c.segs:
                g.wcet *= 1000
    b, (wcrt, sched, status, _) = run([s])
    assert status[0] == 0 and sched[0] == 1
    assert wcrt.tolist() == [x * 1000 for x in GOLD["two_chains_one_executor"]["R"]]
    assert max(ch.T for ch in s.chains) > (1 << 31)
