"""Run the product kernels under the host warp emulator (libpaam_emu.so) and compare with the oracle.
DEBUGGING AID: python tools/warp_emu/check.py [analyze|des] ..."""
import ctypes
import os
import random
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from gen.inputs import MS, config2_params, config3_params, flatten, generate_host, make_params  # noqa
from oracle import oracle as O  # noqa
from paper_2404_06452_b200.paam import Batch, PaamBatch, compact_dict  # noqa  (only for the batch struct marshalling)

L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("PAAM_EMU_LIB", "libpaam_emu.so")))
vp = ctypes.c_void_p
L.emu_pack.argtypes = [vp, vp, vp, vp, vp]
L.emu_wide.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int]
L.emu_analyze.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, vp, vp, vp]
L.emu_simulate.argtypes = [vp, vp, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, vp]
L.emu_record_bytes.restype = ctypes.c_uint32
L.emu_fused.argtypes = [vp, vp, vp, vp, vp, vp, vp, ctypes.c_int]


def compact_struct(hb):
    """A paam_batch carrying the compact (paam_batch32) arrays of host batch hb, as paam_pack_analyze32
    builds it; returns (struct, arrays kept alive), or None if hb does not fit the compact layout."""
    d = {name: hb.arrays.get(name) for name in hb.arrays}
    d.update(n_sets=hb.c.n_sets, n_bins=hb.c.n_bins, comm_cost=hb.c.comm_cost, flags=hb.c.flags)
    try:
        c = compact_dict(d)
    except ValueError:
        return None
    b = PaamBatch()
    ctypes.memmove(ctypes.addressof(b), ctypes.addressof(hb.c), ctypes.sizeof(b))
    ptr = lambda a: None if a is None or a.size == 0 else a.ctypes.data
    for name in ("chain_T", "chain_D", "cb_exec", "seg_wcet", "accel_eps", "accel_kappa"):
        setattr(b, name, ptr(c[name]))
    b.seg_kind, b.seg_accel, b.seg_unit = ptr(c["seg_meta"]), None, None
    return b, c


def emu_run(batch, horizon=None, seed=0, first=0, fifo=False):
    hb = Batch.from_host(batch)
    n = hb.n_sets
    rec = np.zeros((max(n, 1), L.emu_record_bytes()), np.uint8)
    st = np.zeros(max(n, 1), np.int32)
    wl = np.zeros(max(n, 1), np.uint32)  # sets handed over to the u64 path (wide.cu)
    wc = np.zeros(2, np.uint32)  # wide count, work ticket
    L.emu_pack(ctypes.addressof(hb.c), rec.ctypes.data, st.ctypes.data, wl.ctypes.data, wc.ctypes.data)
    L.emu_wide(ctypes.addressof(hb.c), wl.ctypes.data, wc.ctypes.data, st.ctypes.data, None, None, None, None, 0)
    wide = lambda w_, s_, b_: L.emu_wide(ctypes.addressof(hb.c), wl.ctypes.data, wc.ctypes.data, None, w_, s_, b_, None, 0)
    nch = max(hb.c.n_chains, 1)
    w = np.zeros(nch, np.uint64)
    sc = np.zeros(max(n, 1), np.uint8)
    bins = np.zeros(max(2 * hb.c.n_bins, 1), np.int64)
    L.emu_analyze(rec.ctypes.data, n, hb.c.comm_cost, hb.c.flags, hb.c.n_bins if hb.c.set_bin else 0,
                  w.ctypes.data, sc.ctypes.data, bins.ctypes.data if hb.c.set_bin else None)
    wide(w.ctypes.data, sc.ctypes.data, bins.ctypes.data if hb.c.set_bin else None)
    out = dict(status=st[:n], wcrt=w[:hb.c.n_chains], sched=sc[:n], bins=bins[:2 * hb.c.n_bins])
    # PAAM_FLAG_VERDICT_ONLY (0x4): no WCRTs, early exit at the first CRITICAL miss; same verdicts / bins
    sv = np.zeros(max(n, 1), np.uint8)
    bv = np.zeros(max(2 * hb.c.n_bins, 1), np.int64)
    L.emu_analyze(rec.ctypes.data, n, hb.c.comm_cost, hb.c.flags | 0x4, hb.c.n_bins if hb.c.set_bin else 0,
                  None, sv.ctypes.data, bv.ctypes.data if hb.c.set_bin else None)
    wide(None, sv.ctypes.data, bv.ctypes.data if hb.c.set_bin else None)
    out.update(sched_v=sv[:n], bins_v=bv[:2 * hb.c.n_bins])
    # the fused kernel (paam_pack_analyze): full mode and verdict-only
    fst = np.full(max(n, 1), -9, np.int32)
    fw = np.zeros(nch, np.uint64)
    fs = np.zeros(max(n, 1), np.uint8)
    fb = np.zeros(max(2 * hb.c.n_bins, 1), np.int64)
    fl, fc = np.zeros(max(n, 1), np.uint32), np.zeros(2, np.uint32)  # wide count, work ticket
    L.emu_fused(ctypes.addressof(hb.c), fl.ctypes.data, fc.ctypes.data, fst.ctypes.data, fw.ctypes.data, fs.ctypes.data,
                fb.ctypes.data if hb.c.set_bin else None, 0)
    L.emu_wide(ctypes.addressof(hb.c), fl.ctypes.data, fc.ctypes.data, fst.ctypes.data, fw.ctypes.data, fs.ctypes.data,
               fb.ctypes.data if hb.c.set_bin else None, None, 0)
    # the same through the compact batch (paam_pack_analyze32's kernels), when the batch fits it
    cs = compact_struct(hb)
    if cs is not None:
        cst = np.full(max(n, 1), -9, np.int32)
        cw = np.zeros(nch, np.uint64)
        csc = np.zeros(max(n, 1), np.uint8)
        cbn = np.zeros(max(2 * hb.c.n_bins, 1), np.int64)
        cl, cc = np.zeros(max(n, 1), np.uint32), np.zeros(2, np.uint32)
        L.emu_fused(ctypes.addressof(cs[0]), cl.ctypes.data, cc.ctypes.data, cst.ctypes.data, cw.ctypes.data,
                    csc.ctypes.data, cbn.ctypes.data if hb.c.set_bin else None, 1)
        L.emu_wide(ctypes.addressof(cs[0]), cl.ctypes.data, cc.ctypes.data, cst.ctypes.data, cw.ctypes.data,
                   csc.ctypes.data, cbn.ctypes.data if hb.c.set_bin else None, None, 1)
        out_c = dict(c_status=cst[:n], c_wcrt=cw[:hb.c.n_chains], c_sched=csc[:n], c_bins=cbn[:2 * hb.c.n_bins])
    else:
        out_c = {}
    vb = Batch.from_host(dict(batch, flags=batch.get("flags", 0) | 0x4))
    fsv = np.zeros(max(n, 1), np.uint8)
    fbv = np.zeros(max(2 * hb.c.n_bins, 1), np.int64)
    fc[:] = 0
    L.emu_fused(ctypes.addressof(vb.c), fl.ctypes.data, fc.ctypes.data, None, None, fsv.ctypes.data,
                fbv.ctypes.data if hb.c.set_bin else None, 0)
    L.emu_wide(ctypes.addressof(vb.c), fl.ctypes.data, fc.ctypes.data, None, None, fsv.ctypes.data,
               fbv.ctypes.data if hb.c.set_bin else None, None, 0)
    out.update(f_status=fst[:n], f_wcrt=fw[:hb.c.n_chains], f_sched=fs[:n], f_bins=fb[:2 * hb.c.n_bins],
               f_sched_v=fsv[:n], f_bins_v=fbv[:2 * hb.c.n_bins], **out_c)
    if horizon is not None:
        from paper_2404_06452_b200.paam import PaamSimOut
        a = {k: np.zeros(nch, np.uint64) for k in ("resp", "count", "misses", "drops")}
        dig = np.zeros(max(n, 1), np.uint64)
        viol = np.zeros(1, np.int64)
        status = np.full(max(n, 1), -1, np.int32)
        o = PaamSimOut()
        for k, v in a.items():
            setattr(o, k, v.ctypes.data)
        o.digest, o.status, o.violations = dig.ctypes.data, status.ctypes.data, viol.ctypes.data
        o.bound = None if fifo else w.ctypes.data
        L.emu_simulate(ctypes.addressof(hb.c), rec.ctypes.data, n, horizon, seed, first, 1 if fifo else 0,
                       ctypes.addressof(o))
        out.update({k: v[:hb.c.n_chains] for k, v in a.items()})
        out.update(digest=dig[:n], violations=int(viol[0]), sim_status=status[:n])
    return out


def compare(batch, horizon=None, seed=0, first=0, label="", fifo=False):
    e = emu_run(batch, horizon, seed, first, fifo)
    ow, osch, ost, ob = O.analyze(batch)
    ok = np.array_equal(ost, e["status"]) and np.array_equal(ow, e["wcrt"]) and np.array_equal(osch, e["sched"])
    ok = ok and np.array_equal(osch, e["sched_v"]) and np.array_equal(e["bins"], e["bins_v"])
    okf = (np.array_equal(ost, e["f_status"]) and np.array_equal(ow, e["f_wcrt"]) and np.array_equal(osch, e["f_sched"])
           and np.array_equal(osch, e["f_sched_v"]) and np.array_equal(e["bins"], e["f_bins"])
           and np.array_equal(e["bins"], e["f_bins_v"]))
    if not okf:
        bad = np.nonzero(ow != e["f_wcrt"])[0][:5]
        print(f"  FUSED MISMATCH status o={ost[:8]} f={e['f_status'][:8]} wcrt bad {bad} o={ow[bad]} f={e['f_wcrt'][bad]}")
    ok = ok and okf
    if "c_wcrt" in e:  # the compact batch gives the u64 batch's results
        okc = all(np.array_equal(e["f_" + k], e["c_" + k]) for k in ("status", "wcrt", "sched", "bins"))
        if not okc:
            print(f"  COMPACT MISMATCH status f={e['f_status'][:8]} c={e['c_status'][:8]}")
        ok = ok and okc
    msg = [f"{label}: analyze {'OK' if ok else 'MISMATCH'}" + (" (+compact)" if "c_wcrt" in e else "")]
    if not ok:
        bad = np.nonzero(ow != e["wcrt"])[0][:5]
        msg.append(f"  status o={ost[:8]} e={e['status'][:8]} wcrt bad idx {bad} o={ow[bad]} e={e['wcrt'][bad]}")
    if horizon is not None:
        o = O.simulate(batch, horizon, seed=seed, first_index=first, bound=None if fifo else e["wcrt"], nthreads=8, fifo=fifo)
        # sets whose oracle backlog exceeds the device's 4 slots are stopped (PAAM_SIM_BACKLOG = 2) and
        # excluded; every other set must agree exactly (and then the violation counts agree as well
        # unless a stopped set had violations in the oracle's full run)
        off = batch["set_chain_off"].astype(np.int64)
        m = np.diff(off)
        nz = m > 0
        over = np.zeros(len(m), bool)
        if nz.any():
            pk = np.maximum.reduceat(o["peak_live"], (np.cumsum(m) - m)[nz])
            over[nz] = pk > 4
        full = ~np.repeat(over, m)
        ok2 = np.array_equal(e["sim_status"] == 2, over) and not (e["sim_status"] == 3).any()
        for k in ("resp", "count", "misses", "drops"):
            ok2 = ok2 and np.array_equal(o[k][full], e[k][full])
        ok2 = ok2 and np.array_equal(o["digest"][~over], e["digest"][~over])
        msg.append(f"  des {'OK' if ok2 else 'MISMATCH'}")
        if not ok2:
            msg.append(f"  resp o={o['resp'][:8]} e={e['resp'][:8]}\n  count o={o['count'][:8]} e={e['count'][:8]}"
                       f"\n  dig o={o['digest'][:4]} e={e['digest'][:4]} viol o={o['violations']} e={e['violations']}")
        ok = ok and ok2
    print("\n".join(msg), flush=True)
    return ok


if __name__ == "__main__":
    from tests.ref_scan import random_small_system
    import tests.test_oracle_pins as P
    what = sys.argv[1] if len(sys.argv) > 1 else "des"
    systems = {"two": P.two_chain_accel_system(kappa=100_000, buckets=2), "appb": P.app_b_two_chains(),
               "a10": P.a10_system(), "cs3": P.cs3_system(6), "cs3n1": P.cs3_system(1)}
    for nm, s in systems.items():
        compare(flatten([s], comm_cost=0), horizon=500 * MS if what == "des" else None, seed=1, label=nm)
    rng = random.Random(1)
    for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
        s = random_small_system(rng, max_chains=5, tmax=50)
        if not compare(flatten([s], comm_cost=1), horizon=300 if what == "des" else None, seed=i % 3, label=f"rand{i}"):
            print(s)
            break
