"""Run the GPU DES on small systems one at a time (each in a subprocess with a timeout) and compare
with the oracle; prints the first mismatch / hang.  Debug aid."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
from tests.test_gpu_des import gpu_sim
from oracle import oracle as O
from gen.inputs import flatten
import tests.test_oracle_pins as P
import random
from tests.ref_scan import random_small_system
which = sys.argv[1]
if which.startswith("rand"):
    rng = random.Random(int(which[4:])); s = random_small_system(rng, max_chains=4, tmax=40); hz = 200
else:
    s = {"two": lambda: P.two_chain_accel_system(kappa=100_000, buckets=2), "appb": P.app_b_two_chains,
         "cs3": lambda: P.cs3_system(6), "cs3n1": lambda: P.cs3_system(1), "a10": P.a10_system}[which](); hz = 500_000_000
b = flatten([s], comm_cost=0)
for seed in (0, 1):
    g = gpu_sim(b, hz, seed)
    o = O.simulate(b, hz, seed=seed, bound=g["bound"])
    ok = np.array_equal(o["resp"], g["resp"]) and np.array_equal(o["count"], g["count"]) and np.array_equal(o["digest"], g["digest"])
    print(json.dumps(dict(which=which, seed=seed, ok=bool(ok), o=o["resp"].tolist(), g=g["resp"].tolist(),
                          oc=o["count"].tolist(), gc=g["count"].tolist(), od=o["digest"].tolist(), gd=g["digest"].tolist())), flush=True)
''' % ROOT

names = ["two", "appb", "a10", "cs3", "cs3n1"] + [f"rand{i}" for i in range(12)]
for nm in names:
    try:
        r = subprocess.run([sys.executable, "-c", CHILD, nm], capture_output=True, text=True, timeout=60)
        print(nm, "rc", r.returncode, r.stdout.strip()[-800:], r.stderr.strip()[-400:], flush=True)
    except subprocess.TimeoutExpired:
        print(nm, "TIMEOUT", flush=True)
