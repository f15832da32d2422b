"""Small end-to-end run of every kernel (generate, pack, analyze, pack_analyze, simulate PAAM/FIFO, admit)
for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os, random, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from gen.inputs import MS, config2_params, config3_params, flatten, make_params
from paper_2404_06452_b200 import paam
from tests.ref_scan import random_small_system

dev = torch.device("cuda")
for gp, seed in ((config3_params(), 3), (config2_params(0.25), 2), (make_params(exec_mode=1, xexec_frac=0.5, spin_frac=0.5), 5)):
    pp = paam.PaamGenParams.from_buffer_copy(bytes(gp))
    n = 5000
    raw = paam.Raw(pp, seed, 0, n)
    sets = paam.Sets(raw)
    w = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    sc = torch.empty(n, dtype=torch.uint8, device=dev)
    bins = torch.zeros(2 * gp.n_bins, dtype=torch.int64, device=dev)
    sets.pack_analyze(raw, w, sc, bins)
    sets.analyze(w, sc, bins)
    resp = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
    dig = torch.empty(n, dtype=torch.int64, device=dev)
    viol = torch.zeros(1, dtype=torch.int64, device=dev)
    sets.simulate(500 * MS, 1, resp, None, dig, w, viol, n=64)
    sets.simulate(500 * MS, 1, resp, None, dig, None, None, n=64, fifo=True)
    dec = torch.empty(n, dtype=torch.int32, device=dev)
    sets.admit(dec)
    torch.cuda.synchronize()
rng = random.Random(3)
b = paam.Batch.from_host(flatten([random_small_system(rng) for _ in range(300)], comm_cost=1, flags=3))
sets = paam.Sets(b)
w = torch.empty(b.c.n_chains, dtype=torch.int64, device=dev)
sets.analyze(w, None, None)
resp = torch.empty(b.c.n_chains, dtype=torch.int64, device=dev)
sets.simulate(300, 2, resp, None, None, w, None)
torch.cuda.synchronize()
print("sanitize run ok", paam.kernel_launches())
