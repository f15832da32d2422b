"""The compact batch's host-side marshalling (paam.compact_dict, include/paam.h paam_batch32): the packed
segment byte is kind | accel << 1 | unit << 3 (CPU segments carry 0), times and executors keep their
values in the narrower types, and a value the layout cannot hold is refused rather than truncated.  CPU
only: the GPU parity of paam_pack_analyze32 is tests/test_gpu_parity.py."""
import numpy as np
import pytest

from gen.inputs import MS, System, acc, cb, cpu, flatten
from paper_2404_06452_b200.paam import BATCH32_ARRAYS, compact_dict


def _batch():
    s = System()
    g = s.accel(buckets=6, units=3, server_core=0)
    t = s.accel(buckets=1, units=1, server_core=0)
    x = s.executor(core=1)
    y = s.executor(core=2)
    s.chain(T=100 * MS, prio=2, cbs=[cb(x, cpu(1 * MS), acc(g, 2 * MS, unit=2), cpu(3 * MS)), cb(y, acc(t, 4 * MS))])
    s.chain(T=50 * MS, prio=1, cbs=[cb(y, cpu(5 * MS))])
    return flatten([s], comm_cost=7)


def test_compact_layout_and_values():
    b = _batch()
    c = compact_dict(b)
    assert [k for k, _ in BATCH32_ARRAYS] == [k for k in c if k in dict(BATCH32_ARRAYS)]
    assert c["seg_meta"].tolist() == [0, 1 | (0 << 1) | (2 << 3), 0, 1 | (1 << 1) | (0 << 3), 0]
    for k in ("chain_T", "chain_D", "seg_wcet", "accel_eps", "accel_kappa"):
        assert c[k].dtype == np.uint32 and np.array_equal(c[k].astype(np.uint64), b[k].astype(np.uint64))
    assert c["cb_exec"].dtype == np.uint8 and c["cb_exec"].tolist() == b["cb_exec"].tolist()
    for k in ("set_chain_off", "chain_cb_off", "cb_seg_off", "chain_prio", "exec_prio"):
        assert np.array_equal(c[k], b[k])
    assert c["comm_cost"] == 7


def test_compact_refuses_what_it_cannot_hold():
    b = _batch()
    big = dict(b, chain_T=b["chain_T"].astype(np.uint64) + (1 << 32))
    with pytest.raises(ValueError):
        compact_dict(big)
    k = b["seg_kind"].copy()
    k[0] = 2  # undefined kind: the compact byte has one kind bit
    with pytest.raises(ValueError):
        compact_dict(dict(b, seg_kind=k))
    a = b["seg_accel"].copy()
    a[1] = 4  # accelerator index beyond the 2-bit field
    with pytest.raises(ValueError):
        compact_dict(dict(b, seg_accel=a))
    # a CPU segment's accelerator / unit fields do not matter (zeroed, never refused)
    a = b["seg_accel"].copy()
    a[0] = 200
    assert compact_dict(dict(b, seg_accel=a))["seg_meta"][0] == 0
