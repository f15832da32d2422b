"""Seeded synthetic inputs shared by the oracle and the CUDA path (input generation only).

Holds no arithmetic of the analysed method: it builds chain sets in the paper's system model
(PAPER.md:101-142 -- callbacks of alternating CPU/accelerator segments, chains with period,
deadline, unique priority and class, executors on cores with process priorities and a wait
policy, PAAM accelerator servers with n buckets) and flattens them into the CSR arrays that both
`include/paam.h` (paam_batch) and `oracle/oracle.h` (or_batch) describe.

Two sources:
  * `System` -- hand-built sets (the paper's case studies, worked examples, tests);
  * `generate_host` -- the counter-based generator of gen/paam_gen.h run on the
    host through gen/libpaam_gen.so; the device runs the very same header in paam_generate.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MS = 1_000_000
US = 1_000

CPU, ACCEL = 0, 1
CRITICAL, BEST_EFFORT = 0, 1
SUSPEND, SPIN = 0, 1


# ----------------------------------------------------------------------------------------------
# Hand-built systems
@dataclass
class Seg:
    kind: int
    wcet: int
    accel: int = 0
    unit: int = 0


def cpu(wcet: int) -> Seg:
    return Seg(CPU, int(wcet))


def acc(accel: int, wcet: int, unit: int = 0) -> Seg:
    return Seg(ACCEL, int(wcet), accel, unit)


@dataclass
class Callback:
    exec: int
    segs: list


@dataclass
class Chain:
    T: int
    D: int
    prio: int
    cls: int
    cbs: list


@dataclass
class System:
    chains: list = field(default_factory=list)
    execs: list = field(default_factory=list)  # (core, prio, wait)
    accels: list = field(default_factory=list)  # (buckets, units, server_core, eps, kappa)
    bin: int = 0

    def accel(self, buckets=1, units=1, server_core=0, eps=0, kappa=0) -> int:
        self.accels.append((buckets, units, server_core, int(eps), int(kappa)))
        return len(self.accels) - 1

    def executor(self, core, prio=1, wait=SUSPEND) -> int:
        self.execs.append((core, prio, wait))
        return len(self.execs) - 1

    def chain(self, T, D=None, prio=1, cls=CRITICAL, cbs=()) -> int:
        self.chains.append(Chain(int(T), int(T if D is None else D), int(prio), cls, list(cbs)))
        return len(self.chains) - 1


def cb(exec_idx: int, *segs: Seg) -> Callback:
    return Callback(exec_idx, list(segs))


def flatten(systems, comm_cost=100 * US, flags=0, n_bins=0) -> dict:
    """CSR arrays (numpy) of a list of Systems, in the layout of paam_batch / or_batch."""
    set_chain_off, set_exec_off, set_accel_off = [0], [0], [0]
    T, D, P, C, chain_cb_off = [], [], [], [], [0]
    cb_exec, cb_seg_off = [], [0]
    kind, wcet, sacc, sunit = [], [], [], []
    ecore, eprio, ewait = [], [], []
    ab, au, asc, aeps, akap = [], [], [], [], []
    bins = []
    for s in systems:
        for ch in s.chains:
            T.append(ch.T); D.append(ch.D); P.append(ch.prio); C.append(ch.cls)
            for c in ch.cbs:
                cb_exec.append(c.exec)
                for g in c.segs:
                    kind.append(g.kind); wcet.append(g.wcet); sacc.append(g.accel); sunit.append(g.unit)
                cb_seg_off.append(len(kind))
            chain_cb_off.append(len(cb_exec))
        for (core, prio, wait) in s.execs:
            ecore.append(core); eprio.append(prio); ewait.append(wait)
        for (b, u, sc, e, k) in s.accels:
            ab.append(b); au.append(u); asc.append(sc); aeps.append(e); akap.append(k)
        set_chain_off.append(len(T)); set_exec_off.append(len(ecore)); set_accel_off.append(len(ab))
        bins.append(s.bin)
    u8, u16, u32, u64 = np.uint8, np.uint16, np.uint32, np.uint64
    return dict(
        n_sets=len(systems), n_bins=n_bins, comm_cost=int(comm_cost), flags=int(flags),
        set_chain_off=np.array(set_chain_off, u32), set_exec_off=np.array(set_exec_off, u32),
        set_accel_off=np.array(set_accel_off, u32),
        chain_T=np.array(T, u64), chain_D=np.array(D, u64), chain_prio=np.array(P, u32),
        chain_class=np.array(C, u8), chain_cb_off=np.array(chain_cb_off, u32),
        cb_exec=np.array(cb_exec, u16), cb_seg_off=np.array(cb_seg_off, u32),
        seg_kind=np.array(kind, u8), seg_wcet=np.array(wcet, u64), seg_accel=np.array(sacc, u8),
        seg_unit=np.array(sunit, u8),
        exec_core=np.array(ecore, u8), exec_prio=np.array(eprio, u32), exec_wait=np.array(ewait, u8),
        accel_buckets=np.array(ab, u8), accel_units=np.array(au, u8), accel_server_core=np.array(asc, u8),
        accel_eps=np.array(aeps, u64), accel_kappa=np.array(akap, u64),
        set_bin=np.array(bins, u32),
    )


# Field order of paam_batch (include/paam.h) and or_batch (oracle/oracle.h): both bindings build
# their ctypes Structure from this list.
ARRAY_FIELDS = [
    ("set_chain_off", np.uint32), ("set_exec_off", np.uint32), ("set_accel_off", np.uint32),
    ("chain_T", np.uint64), ("chain_D", np.uint64), ("chain_prio", np.uint32), ("chain_class", np.uint8),
    ("chain_cb_off", np.uint32), ("cb_exec", np.uint16), ("cb_seg_off", np.uint32),
    ("seg_kind", np.uint8), ("seg_wcet", np.uint64), ("seg_accel", np.uint8), ("seg_unit", np.uint8),
    ("exec_core", np.uint8), ("exec_prio", np.uint32), ("exec_wait", np.uint8),
    ("accel_buckets", np.uint8), ("accel_units", np.uint8), ("accel_server_core", np.uint8),
    ("accel_eps", np.uint64), ("accel_kappa", np.uint64),
    ("set_bin", np.uint32),
]


def totals(batch: dict) -> dict:
    return dict(n_chains=int(batch["set_chain_off"][-1]), n_cbs=int(batch["chain_cb_off"][-1]),
                n_segs=int(batch["cb_seg_off"][-1]), n_execs=int(batch["set_exec_off"][-1]),
                n_accels=int(batch["set_accel_off"][-1]))


def slice_sets(batch: dict, lo: int, hi: int) -> dict:
    """Sets [lo, hi) of a host batch as a new, rebased batch (for chunked oracle runs)."""
    sc, se, sa = batch["set_chain_off"], batch["set_exec_off"], batch["set_accel_off"]
    c0, c1, e0, e1, a0, a1 = int(sc[lo]), int(sc[hi]), int(se[lo]), int(se[hi]), int(sa[lo]), int(sa[hi])
    cco = batch["chain_cb_off"]
    b0, b1 = int(cco[c0]), int(cco[c1])
    cso = batch["cb_seg_off"]
    g0, g1 = int(cso[b0]), int(cso[b1])
    out = dict(n_sets=hi - lo, n_bins=batch["n_bins"], comm_cost=batch["comm_cost"], flags=batch["flags"])
    out["set_chain_off"] = (sc[lo:hi + 1] - c0).astype(np.uint32)
    out["set_exec_off"] = (se[lo:hi + 1] - e0).astype(np.uint32)
    out["set_accel_off"] = (sa[lo:hi + 1] - a0).astype(np.uint32)
    for k in ("chain_T", "chain_D", "chain_prio", "chain_class"):
        out[k] = batch[k][c0:c1]
    out["chain_cb_off"] = (cco[c0:c1 + 1] - b0).astype(np.uint32)
    out["cb_exec"] = batch["cb_exec"][b0:b1]
    out["cb_seg_off"] = (cso[b0:b1 + 1] - g0).astype(np.uint32)
    for k in ("seg_kind", "seg_wcet", "seg_accel", "seg_unit"):
        out[k] = batch[k][g0:g1]
    for k in ("exec_core", "exec_prio", "exec_wait"):
        out[k] = batch[k][e0:e1]
    for k in ("accel_buckets", "accel_units", "accel_server_core", "accel_eps", "accel_kappa"):
        out[k] = batch[k][a0:a1]
    out["set_bin"] = batch["set_bin"][lo:hi] if batch.get("set_bin") is not None else None
    return out


# ----------------------------------------------------------------------------------------------
# Generator parameters (layout of pg_params == paam_gen_params)
class GenParams(ctypes.Structure):
    _fields_ = [
        ("m_lo", ctypes.c_uint32), ("m_hi", ctypes.c_uint32), ("cbs_per_chain", ctypes.c_uint32),
        ("n_bins", ctypes.c_uint32), ("u_lo_q20", ctypes.c_uint32), ("u_step_q20", ctypes.c_uint32),
        ("ratio_acc", ctypes.c_uint32), ("ratio_cpu", ctypes.c_uint32),
        ("period_min_us", ctypes.c_uint32), ("period_span_q12", ctypes.c_uint32),
        ("exec_mode", ctypes.c_uint32), ("n_cores", ctypes.c_uint32), ("n_exec", ctypes.c_uint32),
        ("n_accel", ctypes.c_uint32),
        ("buckets", ctypes.c_uint32 * 4), ("units", ctypes.c_uint32 * 4),
        ("eps", ctypes.c_uint64 * 4), ("kappa", ctypes.c_uint64 * 4),
        ("be_frac_q16", ctypes.c_uint32), ("spin_frac_q16", ctypes.c_uint32),
        ("cpu_only_frac_q16", ctypes.c_uint32), ("xexec_frac_q16", ctypes.c_uint32),
        ("rm_priorities", ctypes.c_uint32), ("_pad", ctypes.c_uint32),
    ]


def q20(x: float) -> int:
    return int(round(x * (1 << 20)))


def q16(x: float) -> int:
    return int(round(x * (1 << 16)))


def span_q12(t_min_us: int, t_max_us: int) -> int:
    import math
    return int(math.floor(4096 * math.log2(t_max_us / t_min_us)))


def make_params(**kw) -> GenParams:
    """Defaults = SURVEY.md §8(d) config 3 (1M sets): m in [8,16], k=4, 9 bins U=0.1..0.9, 1:1,
    T log-uniform in [100 ms, 1 s], mode A on 4 client cores, GPU-like n=6 (kappa 130 us) +
    TPU-like n=1, eps 391 us, 25% BE, 25% SPIN."""
    d = dict(m_lo=8, m_hi=16, cbs_per_chain=4, n_bins=9, u_lo=0.1, u_step=0.1, ratio_acc=1, ratio_cpu=1,
             t_min_us=100_000, t_max_us=1_000_000, exec_mode=0, n_cores=4, n_exec=4,
             accels=((6, 1, 391 * US, 130 * US), (1, 1, 391 * US, 130 * US)),
             be_frac=0.25, spin_frac=0.25, cpu_only_frac=0.0, xexec_frac=0.0, rm=False)
    d.update(kw)
    p = GenParams()
    p.m_lo, p.m_hi, p.cbs_per_chain, p.n_bins = d["m_lo"], d["m_hi"], d["cbs_per_chain"], d["n_bins"]
    p.u_lo_q20, p.u_step_q20 = q20(d["u_lo"]), q20(d["u_step"])
    p.ratio_acc, p.ratio_cpu = d["ratio_acc"], d["ratio_cpu"]
    p.period_min_us, p.period_span_q12 = d["t_min_us"], span_q12(d["t_min_us"], d["t_max_us"])
    p.exec_mode, p.n_cores, p.n_exec = d["exec_mode"], d["n_cores"], d["n_exec"]
    p.n_accel = len(d["accels"])
    for i, (b, u, e, k) in enumerate(d["accels"]):
        p.buckets[i], p.units[i], p.eps[i], p.kappa[i] = b, u, e, k
    p.be_frac_q16, p.spin_frac_q16 = q16(d["be_frac"]), q16(d["spin_frac"])
    p.cpu_only_frac_q16, p.xexec_frac_q16 = q16(d["cpu_only_frac"]), q16(d["xexec_frac"])
    p.rm_priorities = 1 if d["rm"] else 0
    return p


# Named workloads (SURVEY.md §8(d) "Configs as concrete inputs")
def config2_params(cpu_only_frac=0.0) -> GenParams:
    """10k sets: m in [4,12], k=4, 1 accelerator n=6, executor mode B (4 executors on 4 cores)."""
    return make_params(m_lo=4, m_hi=12, exec_mode=1, n_exec=4, accels=((6, 1, 391 * US, 130 * US),),
                       be_frac=0.0, spin_frac=0.0, cpu_only_frac=cpu_only_frac)


def config3_params() -> GenParams:
    return make_params()


CONFIG_SEEDS = {"config2": 2, "config3": 3, "config4": 4, "config5": 3}


# ----------------------------------------------------------------------------------------------
# Host generator through gen/libpaam_gen.so
_lib = None


def _genlib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "libpaam_gen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        _lib = ctypes.CDLL(path)
        _lib.pg_batch_totals.argtypes = [ctypes.POINTER(GenParams), ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64)]
        _lib.pg_batch_fill.argtypes = [ctypes.POINTER(GenParams), ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_uint32, ctypes.c_void_p]
        assert _lib.pg_params_size() == ctypes.sizeof(GenParams)
    return _lib


def generate_host(params: GenParams, seed: int, first: int, n: int, comm_cost=100 * US, flags=0,
                  pinned_alloc=None) -> dict:
    """Generate sets [first, first+n) on the host.  `pinned_alloc(nbytes) -> np.ndarray[uint8]`
    may supply page-locked storage (for the end-to-end path)."""
    lib = _genlib()
    tot = (ctypes.c_uint64 * 5)()
    rc = lib.pg_batch_totals(ctypes.byref(params), seed, first, n, tot)
    if rc:
        raise ValueError("generator parameters out of range")
    nch, ncb, nsg, nex, nac = (int(x) for x in tot)
    sizes = dict(set_chain_off=n + 1, set_exec_off=n + 1, set_accel_off=n + 1,
                 chain_T=nch, chain_D=nch, chain_prio=nch, chain_class=nch, chain_cb_off=nch + 1,
                 cb_exec=ncb, cb_seg_off=ncb + 1, seg_kind=nsg, seg_wcet=nsg, seg_accel=nsg, seg_unit=nsg,
                 exec_core=nex, exec_prio=nex, exec_wait=nex, accel_buckets=nac, accel_units=nac,
                 accel_server_core=nac, accel_eps=nac, accel_kappa=nac, set_bin=n)
    out = dict(n_sets=n, n_bins=int(params.n_bins), comm_cost=int(comm_cost), flags=int(flags))
    ptrs = []
    for name, dt in ARRAY_FIELDS:
        cnt = max(sizes[name], 1)
        if pinned_alloc is not None:
            raw = pinned_alloc(cnt * np.dtype(dt).itemsize)
            a = raw.view(dt)[:cnt]
        else:
            a = np.empty(cnt, dt)
        out[name] = a[:sizes[name]]
        ptrs.append(a.ctypes.data)
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    rc = lib.pg_batch_fill(ctypes.byref(params), seed, first, n, arr)
    if rc:
        raise RuntimeError("pg_batch_fill failed")
    return out


def with_candidate(s: System, T, prio, cbs, D=None, cls=CRITICAL) -> System:
    """What-if copy of a hand-built system with one more chain (admission control)."""
    import copy
    t = copy.deepcopy(s)
    t.chain(T=T, D=D, prio=prio, cls=cls, cbs=cbs)
    return t


# ----------------------------------------------------------------------------------------------
# The paper's case-study chain sets (configs 1a / 1b of SURVEY.md §8(d)); inputs only.
def case_study_3(buckets: int = 6) -> System:
    """Case Study 3 (SPEC.md:456-457 split): two critical chains T = D = 120 / 220 ms
    and four BE chains T = 52 ms, each one callback CPU 1 ms + GPU 50 ms + CPU 1 ms, six single-threaded
    executors on their own cores, the GPU server on core 0 with n buckets (6 = PAAM's default, P:344;
    1 = TPU-like), eps = 391 us, kappa = 130 us."""
    s = System()
    g = s.accel(buckets=buckets, units=1, server_core=0, eps=391 * US, kappa=130 * US)
    specs = [(120, 6, CRITICAL), (220, 5, CRITICAL), (52, 4, BEST_EFFORT), (52, 3, BEST_EFFORT),
             (52, 2, BEST_EFFORT), (52, 1, BEST_EFFORT)]
    for i, (T, prio, cls) in enumerate(specs):
        x = s.executor(core=1 + i, prio=1, wait=SUSPEND)
        s.chain(T=T * MS, prio=prio, cls=cls, cbs=[cb(x, cpu(1 * MS), acc(g, 50 * MS), cpu(1 * MS))])
    return s


# Config 1b: Case Study 1's SHAPE, with INVENTED numbers: the paper's chain figure is
# missing, so the periods, the CPU WCETs E and the chain lengths below are this
# repository's, labelled as such.  What follows the paper: 8 chains, critical chains 1-6 (chain 1
# highest priority, chain 6 lowest) and BE 1-2 duplicating chains 1 and 3; every callback has one GPU
# segment of A = 10 ms; the critical chains run on four single-threaded executors on cores 2-7, the BE
# chains on their own executors on cores 2-3; the PAAM server with six buckets on core 0.
CS1_SHAPED = [  # (T = D ms, callbacks' CPU WCETs E ms, executor)   -- invented values
    (400, (4, 2), 0), (500, (2, 3, 2), 0), (600, (6, 4), 1), (800, (3, 3), 1), (1000, (5, 2, 3), 2),
    (1200, (4, 6), 3)]


def case_study_1_shaped() -> System:
    """Config 1b (labelled invented numbers, see CS1_SHAPED)."""
    s = System()
    g = s.accel(buckets=6, units=1, server_core=0, eps=391 * US, kappa=130 * US)
    xs = [s.executor(core=2 + i, prio=2, wait=SUSPEND) for i in range(4)]  # critical executors, cores 2-5
    xbe = [s.executor(core=2, prio=1, wait=SUSPEND), s.executor(core=3, prio=1, wait=SUSPEND)]  # BE, cores 2-3

    def callbacks(es, x):
        return [cb(x, cpu(e * MS // 2), acc(g, 10 * MS), cpu(e * MS - e * MS // 2)) for e in es]
    for i, (T, es, xi) in enumerate(CS1_SHAPED):
        s.chain(T=T * MS, prio=8 - i, cls=CRITICAL, cbs=callbacks(es, xs[xi]))
    for j, src in enumerate((0, 2)):  # BE 1 = chain 1, BE 2 = chain 3 (duplicates), lowest priorities
        T, es, _ = CS1_SHAPED[src]
        s.chain(T=T * MS, prio=2 - j, cls=BEST_EFFORT, cbs=callbacks(es, xbe[j]))
    return s
