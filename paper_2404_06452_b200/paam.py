"""Thin ctypes binding of libpaam.so (include/paam.h).  Argument marshalling only.

Every step of the analysis runs in the library's CUDA kernels; this module moves pointers.  There is
no CPU fallback: if libpaam.so is missing or no CUDA device is present the calls raise.
PyTorch is used only to own device memory and streams.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpaam.so")
UNSCHED = (1 << 64) - 1

PAAM_MEM_HOST, PAAM_MEM_DEVICE = 0, 1
PAAM_FLAG_BLOCKING_SOUND = 0x1
PAAM_FLAG_WFD_UNITS = 0x2
PAAM_FLAG_VERDICT_ONLY = 0x4
PAAM_SIM_FIFO_DIRECT = 0x1
SET_STATUS = {0: "OK", 1: "ERANGE", 2: "EDANGLING", 3: "EACCEL", 4: "ESHAPE", 5: "EDUPPRIO",
              6: "EDEADLINE", 7: "ECORE"}

# paam_batch array fields, in declaration order, with their element types.
BATCH_ARRAYS = [
    ("set_chain_off", np.uint32), ("set_exec_off", np.uint32), ("set_accel_off", np.uint32),
    ("chain_T", np.uint64), ("chain_D", np.uint64), ("chain_prio", np.uint32), ("chain_class", np.uint8),
    ("chain_cb_off", np.uint32), ("cb_exec", np.uint16), ("cb_seg_off", np.uint32),
    ("seg_kind", np.uint8), ("seg_wcet", np.uint64), ("seg_accel", np.uint8), ("seg_unit", np.uint8),
    ("exec_core", np.uint8), ("exec_prio", np.uint32), ("exec_wait", np.uint8),
    ("accel_buckets", np.uint8), ("accel_units", np.uint8), ("accel_server_core", np.uint8),
    ("accel_eps", np.uint64), ("accel_kappa", np.uint64),
    ("set_bin", np.uint32),
]
# paam_batch32 (the compact batch) array fields, in declaration order.
BATCH32_ARRAYS = [
    ("set_chain_off", np.uint32), ("set_exec_off", np.uint32), ("set_accel_off", np.uint32),
    ("chain_T", np.uint32), ("chain_D", np.uint32), ("chain_prio", np.uint32), ("chain_class", np.uint8),
    ("chain_cb_off", np.uint32), ("cb_exec", np.uint8), ("cb_seg_off", np.uint32),
    ("seg_meta", np.uint8), ("seg_wcet", np.uint32),
    ("exec_core", np.uint8), ("exec_prio", np.uint32), ("exec_wait", np.uint8),
    ("accel_buckets", np.uint8), ("accel_units", np.uint8), ("accel_server_core", np.uint8),
    ("accel_eps", np.uint32), ("accel_kappa", np.uint32),
    ("set_bin", np.uint32),
]


class PaamBatch(ctypes.Structure):
    _fields_ = ([("n_sets", ctypes.c_uint32), ("mem", ctypes.c_int32)] +
                [(k, ctypes.c_uint32) for k in ("n_chains", "n_cbs", "n_segs", "n_execs", "n_accels", "n_bins")] +
                [(name, ctypes.c_void_p) for name, _ in BATCH_ARRAYS] +
                [("comm_cost", ctypes.c_uint64), ("flags", ctypes.c_uint32), ("_pad", ctypes.c_uint32)])


class PaamBatch32(ctypes.Structure):
    _fields_ = ([("n_sets", ctypes.c_uint32), ("mem", ctypes.c_int32)] +
                [(k, ctypes.c_uint32) for k in ("n_chains", "n_cbs", "n_segs", "n_execs", "n_accels", "n_bins")] +
                [(name, ctypes.c_void_p) for name, _ in BATCH32_ARRAYS] +
                [("comm_cost", ctypes.c_uint64), ("flags", ctypes.c_uint32), ("_pad", ctypes.c_uint32)])


class PaamGenParams(ctypes.Structure):
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


class PaamSimOut(ctypes.Structure):
    _fields_ = [(k, ctypes.c_void_p) for k in ("resp", "count", "misses", "drops", "digest", "status", "bound",
                                              "violations", "witness", "stopped")] + \
               [("max_witness", ctypes.c_uint32), ("_pad", ctypes.c_uint32)]


PAAM_SIM_OK, PAAM_SIM_INVALID, PAAM_SIM_BACKLOG, PAAM_SIM_STEPCAP, PAAM_SIM_WIDE = 0, 1, 2, 3, 4
PAAM_SIM_QCAP = 4


class PaamError(RuntimeError):
    pass


_lib = None
_vp = ctypes.c_void_p


def lib():
    """Load libpaam.so.  Raises if it has not been built: there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PaamError(f"{LIB_PATH} not built (run __graft_entry__.build() or `make -C {HERE}`)")
        L = ctypes.CDLL(LIB_PATH)
        L.paam_generate.argtypes = [ctypes.POINTER(PaamGenParams), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                    ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(_vp), _vp]
        L.paam_regenerate.argtypes = [_vp, ctypes.POINTER(PaamGenParams), ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, _vp]
        L.paam_raw_batch.argtypes = [_vp, ctypes.POINTER(PaamBatch)]
        L.paam_sweep_create.argtypes = [ctypes.c_uint32, ctypes.POINTER(_vp)]
        L.paam_sweep.argtypes = [_vp, ctypes.POINTER(PaamGenParams), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                 ctypes.c_uint64, ctypes.c_uint32, _vp, _vp, _vp]
        L.paam_sweep_free.argtypes = [_vp]
        L.paam_raw_free.argtypes = [_vp]
        L.paam_raw_free.restype = None
        L.paam_pack.argtypes = [ctypes.POINTER(PaamBatch), ctypes.POINTER(_vp), _vp, _vp]
        L.paam_repack.argtypes = [ctypes.POINTER(PaamBatch), _vp, _vp, _vp]
        L.paam_analyze.argtypes = [_vp, ctypes.c_uint32, _vp, _vp, _vp, _vp]
        L.paam_admit.argtypes = [_vp, ctypes.c_uint32, _vp, _vp, _vp]
        L.paam_pack_analyze.argtypes = [ctypes.POINTER(PaamBatch), _vp, _vp, _vp, _vp, _vp, _vp]
        L.paam_pack_analyze32.argtypes = [ctypes.POINTER(PaamBatch32), _vp, _vp, _vp, _vp, _vp, _vp]
        L.paam_simulate.argtypes = [_vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_uint32, ctypes.POINTER(PaamSimOut), _vp]
        L.paam_sets_info.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                                     ctypes.POINTER(ctypes.c_uint32)]
        L.paam_free.argtypes = [_vp]
        L.paam_free.restype = None
        L.paam_strerror.restype = ctypes.c_char_p
        L.paam_last_error.restype = ctypes.c_char_p
        L.paam_kernel_launches.restype = ctypes.c_uint64
        L.paam_record_bytes.restype = ctypes.c_uint32
        L.paam_copy.argtypes = [_vp, _vp, ctypes.c_size_t, _vp]
        L.paam_set_device.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def check(rc: int, what: str):
    if rc != 0:
        L = lib()
        raise PaamError(f"{what}: {L.paam_strerror(rc).decode()} ({rc}): {L.paam_last_error().decode()}")


def set_device_from_torch():
    """Make torch's current CUDA device the library's current device (one process per GPU)."""
    import torch
    if torch.cuda.is_available():  # without a device the next library call fails with PAAM_ECUDA
        check(lib().paam_set_device(torch.cuda.current_device()), "paam_set_device")


def kernel_launches() -> int:
    return int(lib().paam_kernel_launches())


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    return int(getattr(stream, "cuda_stream", stream)) or None


# ---------------------------------------------------------------------------------------------------
class Batch:
    """A paam_batch plus the buffers it points to (kept alive here).

    `arrays`: dict name -> numpy array (host) or torch tensor (device); counts are derived from the
    offset arrays."""

    def __init__(self, arrays: dict, n_sets: int, mem: int, n_bins=0, comm_cost=100_000, flags=0, totals=None):
        self.arrays = arrays
        b = PaamBatch()
        b.n_sets, b.mem, b.n_bins = n_sets, mem, n_bins
        for k, v in (totals or {}).items():
            setattr(b, k, v)
        for name, _ in BATCH_ARRAYS:
            a = arrays.get(name)
            if a is None:
                setattr(b, name, None)
            elif mem == PAAM_MEM_HOST:
                setattr(b, name, a.ctypes.data if a.size else None)
            else:
                setattr(b, name, a.data_ptr() if a.numel() else None)
        b.comm_cost, b.flags = comm_cost, flags
        self.c = b

    @property
    def n_sets(self):
        return self.c.n_sets

    @staticmethod
    def from_host(d: dict) -> "Batch":
        """Host batch from a dict of numpy arrays (the BATCH_ARRAYS names + n_sets/n_bins/comm_cost/flags)."""
        arrays = {}
        for name, dt in BATCH_ARRAYS:
            a = d.get(name)
            if a is not None:
                a = np.ascontiguousarray(a, dtype=dt)
            arrays[name] = a
        tot = dict(n_chains=int(arrays["set_chain_off"][-1]), n_cbs=int(arrays["chain_cb_off"][-1]),
                   n_segs=int(arrays["cb_seg_off"][-1]), n_execs=int(arrays["set_exec_off"][-1]),
                   n_accels=int(arrays["set_accel_off"][-1]))
        n_bins = int(d.get("n_bins", 0))
        if not n_bins:
            arrays["set_bin"] = None
        return Batch(arrays, int(d["n_sets"]), PAAM_MEM_HOST, n_bins, int(d.get("comm_cost", 100_000)),
                     int(d.get("flags", 0)), tot)

    @staticmethod
    def from_host_to_device(d: dict, device="cuda") -> "Batch":
        """Copy a host dict batch into torch device tensors (the 'inputs resident in HBM' setting)."""
        import torch
        h = Batch.from_host(d)
        arrays = {}
        for name, _ in BATCH_ARRAYS:
            a = h.arrays.get(name)
            arrays[name] = None if a is None else torch.from_numpy(a.view(np.uint8).copy()).to(device)
        tot = {k: getattr(h.c, k) for k in ("n_chains", "n_cbs", "n_segs", "n_execs", "n_accels")}
        return Batch(arrays, h.c.n_sets, PAAM_MEM_DEVICE, h.c.n_bins, h.c.comm_cost, h.c.flags, tot)


def compact_dict(d: dict) -> dict:
    """The paam_batch32 arrays of a host dict batch (BATCH_ARRAYS names): 32-bit times, one packed byte
    kind | accel << 1 | unit << 3 per segment, 8-bit callback executors.  Input marshalling only; raises
    ValueError if a value does not fit the compact layout (include/paam.h paam_batch32)."""
    out = {k: d[k] for k in ("n_sets",) if k in d}
    for k in ("n_bins", "comm_cost", "flags"):
        if k in d:
            out[k] = d[k]
    for name, dt in BATCH32_ARRAYS:
        if name == "seg_meta":
            kind = np.asarray(d["seg_kind"], np.uint64)
            acc = np.asarray(d["seg_accel"], np.uint64)
            unit = np.asarray(d["seg_unit"], np.uint64)
            acc = np.where(kind == 1, acc, 0)
            unit = np.where(kind == 1, unit, 0)
            if (kind > 1).any() or (acc > 3).any() or (unit > 7).any():
                raise ValueError("segment kind / accelerator / unit out of the compact range")
            out[name] = (kind | (acc << 1) | (unit << 3)).astype(np.uint8)
            continue
        a = d.get(name)
        if a is None:
            out[name] = None
            continue
        a = np.asarray(a)
        if a.size and int(a.max()) > np.iinfo(dt).max:
            raise ValueError(f"{name}: a value does not fit {np.dtype(dt).name}")
        out[name] = np.ascontiguousarray(a, dtype=dt)
    return out


class Batch32:
    """A paam_batch32 (compact batch) plus the buffers it points to (host numpy or device torch)."""

    def __init__(self, arrays: dict, n_sets: int, mem: int, n_bins=0, comm_cost=100_000, flags=0, totals=None):
        self.arrays = arrays
        b = PaamBatch32()
        b.n_sets, b.mem, b.n_bins = n_sets, mem, n_bins
        for k, v in (totals or {}).items():
            setattr(b, k, v)
        for name, _ in BATCH32_ARRAYS:
            a = arrays.get(name)
            if a is None:
                setattr(b, name, None)
            elif mem == PAAM_MEM_HOST:
                setattr(b, name, a.ctypes.data if a.size else None)
            else:
                setattr(b, name, a.data_ptr() if a.numel() else None)
        b.comm_cost, b.flags = comm_cost, flags
        self.c = b

    @property
    def n_sets(self):
        return self.c.n_sets

    @staticmethod
    def from_host(d: dict, pin=False) -> "Batch32":
        """Host compact batch from a host dict batch (BATCH_ARRAYS names); pin: page-locked copies."""
        c = compact_dict(d)
        arrays = {}
        for name, _ in BATCH32_ARRAYS:
            a = c.get(name)
            if a is not None and pin:
                import torch
                t = torch.from_numpy(a).pin_memory()
                arrays[name + "_pinned"] = t
                a = t.numpy()
            arrays[name] = a
        tot = dict(n_chains=int(c["set_chain_off"][-1]), n_cbs=int(c["chain_cb_off"][-1]),
                   n_segs=int(c["cb_seg_off"][-1]), n_execs=int(c["set_exec_off"][-1]),
                   n_accels=int(c["set_accel_off"][-1]))
        n_bins = int(d.get("n_bins", 0))
        if not n_bins:
            arrays["set_bin"] = None
        return Batch32(arrays, int(d["n_sets"]), PAAM_MEM_HOST, n_bins, int(d.get("comm_cost", 100_000)),
                       int(d.get("flags", 0)), tot)

    @staticmethod
    def from_host_to_device(d: dict, device="cuda") -> "Batch32":
        """A device compact batch (torch tensors) from a host dict batch."""
        import torch
        h = Batch32.from_host(d)
        arrays = {}
        for name, _ in BATCH32_ARRAYS:
            a = h.arrays.get(name)
            arrays[name] = None if a is None else torch.from_numpy(a.view(np.uint8).copy()).to(device)
        tot = {k: getattr(h.c, k) for k in ("n_chains", "n_cbs", "n_segs", "n_execs", "n_accels")}
        return Batch32(arrays, h.c.n_sets, PAAM_MEM_DEVICE, h.c.n_bins, h.c.comm_cost, h.c.flags, tot)


class Raw:
    """Device raw batch produced by paam_generate (§8(a) step 1)."""

    def __init__(self, params: PaamGenParams, seed: int, first: int, n: int, comm_cost=100_000, flags=0, stream=None):
        self.h = _vp()
        set_device_from_torch()
        check(lib().paam_generate(ctypes.byref(params), seed, first, n, comm_cost, flags, ctypes.byref(self.h),
                                  _stream_ptr(stream)), "paam_generate")
        self.c = PaamBatch()
        check(lib().paam_raw_batch(self.h, ctypes.byref(self.c)), "paam_raw_batch")

    def regenerate(self, params: PaamGenParams, seed: int, first: int, n: int, comm_cost=100_000, flags=0,
                   stream=None):
        """paam_regenerate: generate into this handle, reusing its device buffers."""
        check(lib().paam_regenerate(self.h, ctypes.byref(params), seed, first, n, comm_cost, flags,
                                    _stream_ptr(stream)), "paam_regenerate")
        check(lib().paam_raw_batch(self.h, ctypes.byref(self.c)), "paam_raw_batch")

    @property
    def n_sets(self):
        return self.c.n_sets

    def free(self):
        if self.h:
            lib().paam_raw_free(self.h)
            self.h = _vp()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def to_host(self) -> dict:
        """Copy the device raw batch back (tests: GPU generator == host generator, byte for byte)."""
        import torch
        c = self.c
        counts = dict(set_chain_off=c.n_sets + 1, set_exec_off=c.n_sets + 1, set_accel_off=c.n_sets + 1,
                      chain_T=c.n_chains, chain_D=c.n_chains, chain_prio=c.n_chains, chain_class=c.n_chains,
                      chain_cb_off=c.n_chains + 1, cb_exec=c.n_cbs, cb_seg_off=c.n_cbs + 1,
                      seg_kind=c.n_segs, seg_wcet=c.n_segs, seg_accel=c.n_segs, seg_unit=c.n_segs,
                      exec_core=c.n_execs, exec_prio=c.n_execs, exec_wait=c.n_execs,
                      accel_buckets=c.n_accels, accel_units=c.n_accels, accel_server_core=c.n_accels,
                      accel_eps=c.n_accels, accel_kappa=c.n_accels, set_bin=c.n_sets if c.set_bin else 0)
        out = dict(n_sets=c.n_sets, n_bins=c.n_bins, comm_cost=c.comm_cost, flags=c.flags)
        for name, dt in BATCH_ARRAYS:
            ptr = getattr(c, name)
            cnt = counts[name]
            if not ptr or cnt == 0:
                out[name] = np.zeros(0, dt) if name != "set_bin" else None
                continue
            a = np.empty(cnt, dt)
            check(lib().paam_copy(a.ctypes.data, ptr, a.nbytes, None), "paam_copy")
            out[name] = a
        return out


class Sets:
    """Packed device records (paam_sets handle, §8(a) step 2)."""

    def __init__(self, batch, out_status=None, stream=None):
        self.h = _vp()
        c = batch.c
        st = None if out_status is None else (out_status.ctypes.data if isinstance(out_status, np.ndarray)
                                             else out_status.data_ptr())
        set_device_from_torch()
        check(lib().paam_pack(ctypes.byref(c), ctypes.byref(self.h), st, _stream_ptr(stream)), "paam_pack")
        self._refresh()

    def _refresh(self):
        """n_sets / n_chains / n_bins of the batch last packed into the handle (paam_sets_info)."""
        a, b, c = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        check(lib().paam_sets_info(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "paam_sets_info")
        self.n_sets, self.n_chains, self.n_bins = a.value, b.value, c.value

    def repack(self, batch, out_status=None, stream=None):
        st = None if out_status is None else (out_status.ctypes.data if isinstance(out_status, np.ndarray)
                                             else out_status.data_ptr())
        check(lib().paam_repack(ctypes.byref(batch.c), self.h, st, _stream_ptr(stream)), "paam_repack")
        self._refresh()

    def admit(self, out_decision, out_wcrt=None, n=None, stream=None):
        """Batched admission decisions (paam_admit): -1 accept, >= 0 first failing chain, <= -2 invalid."""
        ptr = lambda t: None if t is None else t.data_ptr()
        check(lib().paam_admit(self.h, self.n_sets if n is None else n, ptr(out_decision), ptr(out_wcrt),
                               _stream_ptr(stream)), "paam_admit")

    def pack_analyze(self, batch, out_wcrt=None, out_sched=None, out_bins=None, out_status=None, stream=None):
        """Pipelined repack + analyze (paam_pack_analyze).  Outputs: device tensors or None; for a host batch
        out_wcrt / out_sched may also be host memory (numpy arrays or pinned CPU tensors), copied back chunk
        by chunk; out_status in the batch's memory space (numpy array for a host batch, device tensor for a
        device batch)."""
        ptr = lambda t: None if t is None else (t.ctypes.data if isinstance(t, np.ndarray) else t.data_ptr())
        st = None if out_status is None else (out_status.ctypes.data if isinstance(out_status, np.ndarray)
                                             else out_status.data_ptr())
        if isinstance(batch, Batch32):
            check(lib().paam_pack_analyze32(ctypes.byref(batch.c), self.h, st, ptr(out_wcrt), ptr(out_sched),
                                            ptr(out_bins), _stream_ptr(stream)), "paam_pack_analyze32")
        else:
            check(lib().paam_pack_analyze(ctypes.byref(batch.c), self.h, st, ptr(out_wcrt), ptr(out_sched),
                                          ptr(out_bins), _stream_ptr(stream)), "paam_pack_analyze")
        self._refresh()

    def analyze(self, out_wcrt=None, out_sched=None, out_bins=None, n=None, stream=None):
        """Device tensors (torch) or None; returns nothing (asynchronous on `stream`)."""
        ptr = lambda t: None if t is None else t.data_ptr()
        check(lib().paam_analyze(self.h, self.n_sets if n is None else n, ptr(out_wcrt), ptr(out_sched),
                                 ptr(out_bins), _stream_ptr(stream)), "paam_analyze")

    def simulate(self, horizon, seed, out_resp=None, out_count=None, out_digest=None, bound=None, out_violations=None,
                 first_index=0, n=None, stream=None, fifo=False, out_misses=None, out_drops=None, out_status=None,
                 out_witness=None, out_stopped=None):
        """paam_simulate (device tensors or None).  out_witness: int32 tensor [2*K] of (set, chain) pairs
        of sim > bound, filled first come (needs out_violations)."""
        ptr = lambda t: None if t is None else t.data_ptr()
        o = PaamSimOut()
        for k, t in (("resp", out_resp), ("count", out_count), ("misses", out_misses), ("drops", out_drops),
                     ("digest", out_digest), ("status", out_status), ("bound", bound), ("violations", out_violations),
                     ("witness", out_witness), ("stopped", out_stopped)):
            setattr(o, k, ptr(t))
        o.max_witness = 0 if out_witness is None else out_witness.numel() // 2
        check(lib().paam_simulate(self.h, self.n_sets if n is None else n, horizon, seed, first_index,
                                  PAAM_SIM_FIFO_DIRECT if fifo else 0, ctypes.byref(o), _stream_ptr(stream)),
              "paam_simulate")

    def free(self):
        if self.h:
            lib().paam_free(self.h)
            self.h = _vp()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Sweeper:
    """paam_sweep: generate -> pack -> analyse over device-generated chunks, generation overlapped with
    analysis, no host synchronisation (§8(a) steps 1-6)."""

    def __init__(self, chunk: int = 262_144):
        self.h = _vp()
        set_device_from_torch()
        check(lib().paam_sweep_create(chunk, ctypes.byref(self.h)), "paam_sweep_create")

    def run(self, params: PaamGenParams, seed: int, first: int, n: int, out_sched=None, out_bins=None,
            comm_cost=100_000, flags=0, stream=None):
        ptr = lambda t: None if t is None else t.data_ptr()
        check(lib().paam_sweep(self.h, ctypes.byref(params), seed, first, n, comm_cost, flags, ptr(out_sched),
                               ptr(out_bins), _stream_ptr(stream)), "paam_sweep")

    def free(self):
        if self.h:
            lib().paam_sweep_free(self.h)
            self.h = _vp()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def analyze(batch, stream=None, fused=False):
    """Analyse a batch; returns numpy (wcrt[n_chains] u64, sched[n] u8, status[n] i32, bins).
    fused=False: paam_pack + paam_analyze (records through HBM); fused=True: paam_pack_analyze (one
    fused_kernel launch, the bench's path; a host batch is copied in chunks overlapping the kernel)."""
    import torch
    n = batch.n_sets
    dev = torch.device("cuda")
    host = batch.c.mem == PAAM_MEM_HOST
    mk_status = lambda: np.full(max(n, 1), -9, np.int32) if host else torch.full((max(n, 1),), -9, dtype=torch.int32, device=dev)
    status = mk_status()
    sets = Sets(batch, None if fused else status, stream)
    wcrt = torch.full((max(batch.c.n_chains, 1),), -5, dtype=torch.int64, device=dev)
    sched = torch.full((max(n, 1),), 7, dtype=torch.uint8, device=dev)
    bins = torch.zeros(max(sets.n_bins * 2, 1), dtype=torch.int64, device=dev)
    if fused:
        sets.pack_analyze(batch, wcrt, sched, bins if sets.n_bins else None, out_status=status, stream=stream)
    else:
        sets.analyze(wcrt, sched, bins if sets.n_bins else None, stream=stream)
    torch.cuda.synchronize()
    st = status if isinstance(status, np.ndarray) else status.cpu().numpy()
    out = (wcrt.cpu().numpy().view(np.uint64)[:batch.c.n_chains], sched.cpu().numpy()[:n], st[:n],
           bins.cpu().numpy()[:sets.n_bins * 2])
    sets.free()
    return out
