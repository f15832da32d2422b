import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from gen.inputs import config3_params
from paper_2404_06452_b200 import paam
gp = config3_params(); pp = paam.PaamGenParams.from_buffer_copy(bytes(gp))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4736
raw = paam.Raw(pp, 3, 0, n); sets = paam.Sets(raw)
dev = torch.device("cuda")
w = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev); sets.analyze(w, None, None)
resp = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
dig = torch.empty(n, dtype=torch.int64, device=dev) if os.environ.get("DES_DIGEST") else None
sets.simulate(10_000_000_000, 3, resp, None, dig, w, None)
torch.cuda.synchronize(); print("ok")
