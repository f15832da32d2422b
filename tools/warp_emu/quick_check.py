import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import random, sys
from tools.warp_emu.check import compare
from gen.inputs import *
from tests.ref_scan import random_small_system
from tests.test_gpu_parity import mutate_invalid
import tests.test_oracle_pins as P
rng = random.Random(11)
ok=True
named = [P.two_chain_accel_system(kappa=100_000, buckets=2), P.app_b_two_chains(), P.a10_system(), P.cs3_system(6), P.cs3_system(1), P.spin_system(1), P.spin_system(0), P.lemma3_union_system()]
ok &= compare(flatten(named, comm_cost=0), label="named")
for rep in range(4):
    systems = [random_small_system(rng, max_chains=6, tmax=200) for _ in range(400)]
    ok &= compare(flatten(systems, comm_cost=3, flags=rep), label=f"random flags {rep}")
inv = [mutate_invalid(random_small_system(rng), rng) for _ in range(300)]
ok &= compare(flatten(inv, comm_cost=1), label="invalid sets")
ok &= compare(generate_host(config3_params(), 4, 0, 400), label="config 3 400")
ok &= compare(generate_host(config2_params(cpu_only_frac=0.25), 2, 0, 400), label="config 2")
ok &= compare(generate_host(make_params(exec_mode=1, n_exec=4, xexec_frac=0.5, spin_frac=0.5, cpu_only_frac=0.2), 6, 0, 300), label="modeB")
ok &= compare(generate_host(make_params(accels=((6, 3, 391000, 130000), (1, 2, 391000, 0))), 3, 0, 300), label="5 units")
print("ALL", ok)
# wide sets: random systems with every time scaled past 2^31 ns, mixed with ordinary ones
def scaled(s, f):
    for ch in s.chains:
        ch.T *= f; ch.D *= f
        for c in ch.cbs:
            for g in c.segs: g.wcet *= f
    s.accels = [(bk, u, sc, e * f, k * f) for (bk, u, sc, e, k) in s.accels]
    return s
rng2 = random.Random(5)
mix = []
for i in range(300):
    s = random_small_system(rng2, max_chains=6, tmax=200)
    mix.append(scaled(s, 1 << 26) if i % 2 else s)
for fl in (0, 1, 2):
    ok &= compare(flatten(mix, comm_cost=3 << 20, flags=fl), label=f"wide mix flags {fl}")
print("ALL2", ok)
