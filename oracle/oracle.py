"""ctypes wrapper of the CPU oracle (oracle/liboracle.so).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this module.  The product path (paper_2404_06452_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from gen.inputs import ARRAY_FIELDS, GenParams, totals  # noqa: E402

UNSCHED = (1 << 64) - 1
DMAX = 256


class OrBatch(ctypes.Structure):
    _fields_ = ([("n_sets", ctypes.c_uint32), ("mem", ctypes.c_int32)] +
                [(k, ctypes.c_uint32) for k in ("n_chains", "n_cbs", "n_segs", "n_execs", "n_accels", "n_bins")] +
                [(name, ctypes.c_void_p) for name, _ in ARRAY_FIELDS] +
                [("comm_cost", ctypes.c_uint64), ("flags", ctypes.c_uint32), ("_pad", ctypes.c_uint32)])


class OrDetail(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("n_sub", ctypes.c_uint32), ("n_aseg", ctypes.c_uint32),
                ("sub_chain", ctypes.c_int32 * DMAX), ("sub_exec", ctypes.c_int32 * DMAX)] + \
               [(k, ctypes.c_uint64 * DMAX) for k in ("sub_B", "sub_E", "sub_S", "sub_C", "sub_Hstar", "sub_R", "sub_iters")] + \
               [("aseg_sub", ctypes.c_int32 * DMAX), ("aseg_bucket", ctypes.c_int32 * DMAX)] + \
               [(k, ctypes.c_uint64 * DMAX) for k in ("aseg_Astar", "aseg_LPB", "aseg_H")] + \
               [("mu_literal", ctypes.c_uint64), ("mu_regrouped", ctypes.c_uint64), ("iterations", ctypes.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle`")
        _lib = ctypes.CDLL(path)
        _lib.oracle_analyze_batch.argtypes = [ctypes.POINTER(OrBatch), ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        _lib.oracle_analyze_detail.argtypes = [ctypes.POINTER(OrBatch), ctypes.c_uint32, ctypes.POINTER(OrDetail)]
        _lib.oracle_generate_analyze.argtypes = [ctypes.POINTER(GenParams), ctypes.c_uint64, ctypes.c_uint64,
                                                 ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32,
                                                 ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        _lib.oracle_simulate_batch.argtypes = [ctypes.POINTER(OrBatch), ctypes.c_uint64, ctypes.c_uint64,
                                               ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_int]
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def make_batch(batch: dict) -> OrBatch:
    b = OrBatch()
    b.n_sets = batch["n_sets"]
    b.mem = 0
    for k, v in totals(batch).items():
        setattr(b, k, v)
    b.n_bins = batch.get("n_bins", 0)
    for name, dt in ARRAY_FIELDS:
        a = batch.get(name)
        if a is not None:
            assert a.dtype == dt, (name, a.dtype, dt)
            assert a.flags["C_CONTIGUOUS"]
        setattr(b, name, _ptr(a) if (a is not None and a.size) else (None if a is None else _ptr(np.zeros(1, dt))))
    b.comm_cost = batch.get("comm_cost", 100_000)
    b.flags = batch.get("flags", 0)
    return b


def analyze(batch: dict, nthreads: int = 1):
    """Returns (wcrt[n_chains] u64, sched[n] u8, status[n] i32, bins[n_bins*2] i64)."""
    b = make_batch(batch)
    keep = batch  # noqa: F841  (arrays referenced by raw pointers stay alive)
    n = batch["n_sets"]
    wcrt = np.zeros(max(int(batch["set_chain_off"][-1]), 1), np.uint64)
    sched = np.zeros(max(n, 1), np.uint8)
    status = np.zeros(max(n, 1), np.int32)
    bins = np.zeros(max(batch.get("n_bins", 0) * 2, 1), np.int64)
    rc = lib().oracle_analyze_batch(ctypes.byref(b), _ptr(wcrt), _ptr(sched), _ptr(status), _ptr(bins), nthreads)
    assert rc == 0
    return wcrt[:int(batch["set_chain_off"][-1])], sched[:n], status[:n], bins[:batch.get("n_bins", 0) * 2]


def detail(batch: dict, set_index: int = 0) -> dict:
    b = make_batch(batch)
    d = OrDetail()
    rc = lib().oracle_analyze_detail(ctypes.byref(b), set_index, ctypes.byref(d))
    assert rc == 0, rc
    ns, na = d.n_sub, d.n_aseg
    out = dict(status=d.status, n_sub=ns, n_aseg=na, mu_literal=d.mu_literal, mu_regrouped=d.mu_regrouped,
               iterations=d.iterations)
    for k in ("sub_chain", "sub_exec", "sub_B", "sub_E", "sub_S", "sub_C", "sub_Hstar", "sub_R", "sub_iters"):
        out[k] = list(getattr(d, k))[:ns]
    for k in ("aseg_sub", "aseg_bucket", "aseg_Astar", "aseg_LPB", "aseg_H"):
        out[k] = list(getattr(d, k))[:na]
    return out


def generate_analyze(params: GenParams, seed: int, first: int, n: int, comm_cost=100_000, flags=0,
                     want_wcrt=False, stride=32, nthreads=1):
    """Oracle run straight from the generator.  Returns (wcrt[n, stride] or None, sched, bins, counters)."""
    wcrt = np.full((n, stride), UNSCHED, np.uint64) if want_wcrt else None
    sched = np.zeros(max(n, 1), np.uint8)
    bins = np.zeros(max(params.n_bins * 2, 1), np.int64)
    cnt = np.zeros(3, np.uint64)
    rc = lib().oracle_generate_analyze(ctypes.byref(params), seed, first, n, comm_cost, flags,
                                       _ptr(wcrt), stride, _ptr(sched), _ptr(bins), _ptr(cnt), nthreads)
    assert rc == 0, rc
    return wcrt, sched[:n], bins[:params.n_bins * 2], cnt


def simulate(batch: dict, horizon: int, seed: int = 0, first_index: int = 0, phases=None, bound=None,
             nthreads: int = 1, fifo: bool = False) -> dict:
    """Oracle DES.  Returns dict(resp, count, misses, drops, peak_live per chain; digest per set;
    violations)."""
    b = make_batch(batch)
    nch = int(batch["set_chain_off"][-1])
    n = batch["n_sets"]
    resp = np.zeros(max(nch, 1), np.uint64)
    cnt = np.zeros(max(nch, 1), np.uint64)
    misc = np.zeros(max(3 * nch, 3), np.uint64)
    dig = np.zeros(max(n, 1), np.uint64)
    viol = np.zeros(1, np.int64)
    ph = None if phases is None else np.ascontiguousarray(phases, np.uint64)
    bd = None if bound is None else np.ascontiguousarray(bound, np.uint64)
    rc = lib().oracle_simulate_batch(ctypes.byref(b), horizon, seed, first_index, 1 if fifo else 0, _ptr(ph), _ptr(resp), _ptr(cnt),
                                     _ptr(misc), _ptr(dig), _ptr(bd), _ptr(viol), nthreads)
    assert rc == 0
    misc = misc[:3 * nch].reshape(-1, 3) if nch else np.zeros((0, 3), np.uint64)
    return dict(resp=resp[:nch], count=cnt[:nch], misses=misc[:, 0], drops=misc[:, 1], peak_live=misc[:, 2],
                digest=dig[:n], violations=int(viol[0]))
