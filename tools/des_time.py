"""Time paam_simulate on n config-3-recipe sets (10 s horizon, seed 3), digests on and off (CUDA events,
after one warm-up run).   python tools/des_time.py [n]  -> one JSON line"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from gen.inputs import config3_params
from paper_2404_06452_b200 import paam
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
gp = config3_params(); pp = paam.PaamGenParams.from_buffer_copy(bytes(gp))
raw = paam.Raw(pp, 3, 0, n); sets = paam.Sets(raw)
dev = torch.device("cuda")
w = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev); sets.analyze(w, None, None)
resp = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
dig = torch.empty(n, dtype=torch.int64, device=dev)
out = {"sets": n}
for name, d in (("digest", dig), ("no_digest", None)):
    sets.simulate(10_000_000_000, 3, resp, None, d, w, None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    sets.simulate(10_000_000_000, 3, resp, None, d, w, None)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out[name] = {"ms": round(ms, 1), "sets_per_s": round(n / ms * 1e3)}
print(json.dumps(out))
