"""Shared input generator (gen/paam_gen.h): invariants of the workload recipe."""
import numpy as np

from gen.inputs import config2_params, generate_host, make_params
from oracle import oracle as O


def per_chain_sums(b):
    seg_chain = np.repeat(np.arange(len(b["chain_T"])), np.diff(b["chain_cb_off"]).astype(np.int64))
    seg_cb = np.repeat(np.arange(len(b["cb_exec"])), np.diff(b["cb_seg_off"]).astype(np.int64))
    seg_owner = seg_chain[seg_cb]
    tot = np.bincount(seg_owner, weights=b["seg_wcet"].astype(np.float64), minlength=len(b["chain_T"]))
    accs = np.bincount(seg_owner, weights=(b["seg_wcet"] * (b["seg_kind"] == 1)).astype(np.float64),
                       minlength=len(b["chain_T"]))
    return tot, accs


def test_utilisation_accounting():
    """Sum_c (sum of WCETs / T_c) == U_total of the set's bin, up to ns rounding."""
    p = make_params()
    b = generate_host(p, seed=3, first=0, n=900)
    tot, accs = per_chain_sums(b)
    util = tot / b["chain_T"].astype(np.float64)
    off = b["set_chain_off"]
    for i in range(b["n_sets"]):
        u = util[off[i]:off[i + 1]].sum()
        target = (p.u_lo_q20 + b["set_bin"][i] * p.u_step_q20) / 2 ** 20
        m = off[i + 1] - off[i]
        assert abs(u - target) < 4 * 3 * m * 2.0 / 1e8 + 1e-6 * m, (i, u, target)
    # 1:1 accelerator : CPU split per callback, up to 1 ns per callback
    assert np.all(np.abs(2 * accs - tot) <= 4 * 2 + 1)


def test_shapes_and_validity():
    for p in (make_params(), config2_params(), config2_params(cpu_only_frac=0.25),
              make_params(exec_mode=1, n_exec=4, xexec_frac=0.5)):
        b = generate_host(p, seed=1, first=0, n=400)
        m = np.diff(b["set_chain_off"])
        assert m.min() >= p.m_lo and m.max() <= p.m_hi
        assert np.all(np.diff(b["chain_cb_off"]) == p.cbs_per_chain)
        # priorities unique within each set
        for i in range(0, 400, 7):
            pr = b["chain_prio"][b["set_chain_off"][i]:b["set_chain_off"][i + 1]]
            assert len(set(pr.tolist())) == len(pr)
        _, _, status, _ = O.analyze(b)
        assert (status == 0).all()


def test_same_seed_same_bytes_and_ranges_compose():
    p = make_params()
    a = generate_host(p, seed=9, first=0, n=300)
    b = generate_host(p, seed=9, first=0, n=300)
    for k, v in a.items():
        if isinstance(v, np.ndarray):
            assert np.array_equal(v, b[k])
    # sets are a pure function of (seed, index): a sub-range equals the slice of the full range
    c = generate_host(p, seed=9, first=100, n=50)
    lo, hi = a["set_chain_off"][100], a["set_chain_off"][150]
    assert np.array_equal(c["chain_T"], a["chain_T"][lo:hi])
    assert np.array_equal(c["chain_prio"], a["chain_prio"][lo:hi])


def test_periods_log_uniform_range():
    p = make_params()
    b = generate_host(p, seed=4, first=0, n=2000)
    T = b["chain_T"].astype(np.float64)
    assert T.min() >= 100e6 and T.max() <= 1000e6
    lg = np.log10(T / 1e6)  # ms
    # log-uniform on [2, 3]: each of 4 quarter-decades holds ~25%
    h, _ = np.histogram(lg, bins=4, range=(2, 3))
    assert np.all(np.abs(h / h.sum() - 0.25) < 0.03)


def test_sizes_only_path_matches_full_generator():
    """pg_set_sizes (used to size the CSR batch without generating the sets) == pg_generate_set's sizes."""
    import ctypes
    from gen.inputs import _genlib, config2_params, config3_params
    lib = _genlib()
    lib.pg_sizes_mismatch.restype = ctypes.c_int64
    lib.pg_sizes_mismatch.argtypes = [ctypes.POINTER(type(make_params())), ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint32]
    for p, seed in ((config3_params(), 3), (config2_params(0.25), 2), (make_params(exec_mode=1, xexec_frac=0.5), 8),
                    (make_params(m_lo=1, m_hi=32, cbs_per_chain=2, cpu_only_frac=0.5), 5)):
        assert lib.pg_sizes_mismatch(ctypes.byref(p), seed, 0, 5000) == 0
