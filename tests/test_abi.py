"""The C-ABI library loads and exports every symbol include/paam.h declares (CPU-only checks)."""
import ctypes
import os
import re

import pytest

from paper_2404_06452_b200 import paam

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "paam.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(paam_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(paam.LIB_PATH):
        pytest.skip("libpaam.so not built")
    L = paam.lib()
    names = declared_functions()
    assert len(names) >= 14, names
    for n in names:
        assert hasattr(L, n), n


def test_struct_layouts_match_header():
    # paam_batch: 2 + 6 u32, 23 pointers, u64 + 2 u32
    assert ctypes.sizeof(paam.PaamBatch) == 8 * 4 + 23 * 8 + 8 + 8
    from gen.inputs import GenParams, _genlib
    assert ctypes.sizeof(paam.PaamGenParams) == ctypes.sizeof(GenParams) == _genlib().pg_params_size()
    assert [f[0] for f in paam.PaamGenParams._fields_] == [f[0] for f in GenParams._fields_]


def test_error_strings():
    if not os.path.exists(paam.LIB_PATH):
        pytest.skip("libpaam.so not built")
    L = paam.lib()
    assert L.paam_strerror(0) == b"ok"
    assert L.paam_strerror(-1) == b"invalid argument"


def test_calls_fail_loudly_without_device():
    """No CPU fallback: on a host without a GPU the entry points raise instead of computing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    if not os.path.exists(paam.LIB_PATH):
        pytest.skip("libpaam.so not built")
    from gen.inputs import make_params
    p = paam.PaamGenParams.from_buffer_copy(bytes(make_params()))
    with pytest.raises(paam.PaamError):
        paam.Raw(p, seed=1, first=0, n=4)
    with pytest.raises(paam.PaamError):
        paam.Sweeper(chunk=1024)


def test_null_arguments_rejected():
    if not os.path.exists(paam.LIB_PATH):
        pytest.skip("libpaam.so not built")
    L = paam.lib()
    assert L.paam_pack(None, None, None, None) == -1
    assert L.paam_analyze(None, 0, None, None, None, None) == -1
    assert L.paam_sweep(None, None, 0, 0, 0, 0, 0, None, None, None) == -1
    assert L.paam_sweep_create(0, None) == -1
    assert L.paam_regenerate(None, None, 0, 0, 0, 0, 0, None) == -1


def test_binding_surface():
    """The thin binding exposes every entry point the tests and bench.py call (no GPU needed)."""
    from paper_2404_06452_b200 import paam
    for cls, names in ((paam.Raw, ("regenerate", "free", "to_host")), (paam.Sweeper, ("run", "free")),
                       (paam.Sets, ("repack", "pack_analyze", "analyze", "admit", "simulate", "free")),
                       (paam.Batch, ("from_host", "from_host_to_device"))):
        for nm in names:
            assert callable(getattr(cls, nm, None)), (cls.__name__, nm)
    assert paam.PAAM_FLAG_VERDICT_ONLY == 0x4
