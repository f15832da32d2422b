"""The CUDA kernel sources (pack / analyze / simulate) compiled as host C++ under tools/warp_emu (every
CUDA thread a host thread, warp intrinsics as 32-thread collectives) and run against the oracle, under
AddressSanitizer + UBSan when available.  A CPU-side logic and memory-safety check of the kernel code
(a divergent warp collective deadlocks the emulator; an out-of-bounds shared/global access trips
ASan).  It is NOT a GPU parity claim -- those are the -m gpu tests -- and the product never uses it."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EMU = os.path.join(ROOT, "tools", "warp_emu")

SCRIPT = r'''
import sys, random
sys.path.insert(0, %r)
from tools.warp_emu.check import compare
from gen.inputs import *
from tests.ref_scan import random_small_system
from tests.test_gpu_parity import mutate_invalid
import tests.test_oracle_pins as P
rng = random.Random(4)
ok = True
named = [P.two_chain_accel_system(kappa=100_000, buckets=2), P.app_b_two_chains(), P.a10_system(), P.cs3_system(6), P.cs3_system(1)]
ok &= compare(flatten(named, comm_cost=0), horizon=400 * MS, seed=1, label="worked examples")
systems = [random_small_system(rng, max_chains=5, tmax=60) for _ in range(60)]
ok &= compare(flatten(systems, comm_cost=1, flags=3), horizon=200, seed=2, label="random WFD+sound")
ok &= compare(flatten(systems, comm_cost=1), horizon=200, seed=0, label="random fifo", fifo=True)
inv = [mutate_invalid(random_small_system(rng), rng) for _ in range(200)]
ok &= compare(flatten(inv, comm_cost=1), label="invalid sets")
ok &= compare(generate_host(config3_params(), 3, 0, 40), label="config 3")
print("EMU_OK" if ok else "EMU_FAIL")
''' % ROOT


def _build(asan):
    target = "libpaam_emu_asan.so" if asan else "libpaam_emu.so"
    flags = "-fsanitize=address,undefined -fno-omit-frame-pointer" if asan else ""
    cmd = (f"g++ -O1 -g -std=c++20 -fPIC -pthread -DPAAM_WARP_EMU {flags} -I../../include -shared -o {target} "
           "emu_pack.cpp emu_analyze.cpp emu_simulate.cpp emu_fused.cpp emu_wide.cpp")
    subprocess.run(cmd, shell=True, cwd=EMU, check=True)
    return target


def test_kernels_under_host_emulation():
    try:
        libasan = subprocess.run(["gcc", "-print-file-name=libasan.so"], capture_output=True, text=True).stdout.strip()
        libubsan = subprocess.run(["gcc", "-print-file-name=libubsan.so"], capture_output=True, text=True).stdout.strip()
        asan = os.path.isabs(libasan) and os.path.exists(libasan) and os.path.exists(libubsan)
    except FileNotFoundError:
        pytest.skip("no gcc")
    target = _build(asan)
    env = dict(os.environ, PAAM_EMU_LIB=target, ASAN_OPTIONS="detect_leaks=0:halt_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    if asan:
        env["LD_PRELOAD"] = f"{libasan} {libubsan}"
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "EMU_OK" in r.stdout, r.stdout[-3000:]
    assert "ERROR: AddressSanitizer" not in r.stderr and "runtime error" not in r.stderr, r.stderr[-3000:]
