"""§8(f) experiments on the GPU path: Fig. 12 curve trends, the A10 blocking census and
the PAAM vs FIFO_DIRECT comparison of Case Study 3."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen.inputs import MS, config2_params, flatten, make_params
from oracle import oracle as O
from paper_2404_06452_b200 import experiments as X
from tests.test_oracle_pins import cs3_system


def test_chain_count_curve_non_increasing():
    """Fig. 12(a): schedulability non-increasing in chains per set (<= 2 pp local noise)."""
    pts = X.chain_count_curve([2, 4, 6, 8, 10, 12, 14, 16], trials=1000, u_total=0.6)
    r = [v for _, v in pts]
    for a, b in zip(r, r[1:]):
        assert b <= a + 0.02, pts
    assert r[0] > r[-1] + 0.05, pts


def test_ratio_curve_decreases():
    """Fig. 12(b): the ratio at 7:3 is > 5 pp below the ratio at 1:9."""
    pts = dict(X.ratio_curve(trials=1000, m=8, u_total=0.6))
    assert pts["7:3"] < pts["1:9"] - 0.05, pts


def test_curve_point_matches_oracle():
    gp = make_params(m_lo=8, m_hi=8, n_bins=1, u_lo=0.5, u_step=0.0)
    g = X.schedulable_ratio(gp, 33, 2000)
    _, s, _, _ = O.generate_analyze(gp, 33, 0, 2000, nthreads=8)
    assert g * 2000 == int(s.sum())


def test_blocking_census_sound_variant_never_violated():
    """A10: shared executors with CPU-only callbacks.  The sound bound is never exceeded; the
    as-written count is reported (a census, not an assertion)."""
    gp = config2_params(cpu_only_frac=0.4)
    res = X.blocking_census(gp, seed=2, n=3000, horizon_ns=5_000 * MS)
    assert res["sound"]["violating_chains"] == 0
    assert res["as_written"]["schedulable_sets"] >= res["sound"]["schedulable_sets"]
    print("A10 census", res)


def test_fifo_comparison_case_study_3():
    best = X.fifo_comparison(flatten([cs3_system(6)], comm_cost=0), 3_000 * MS, seeds=range(6))
    assert best["paam"][0] <= best["bound"][0]
    assert best["paam"][0] <= 0.8 * best["fifo"][0]
