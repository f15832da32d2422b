"""One paam_pack (pack_kernel) and one paam_analyze (analyze_kernel) launch on N config-3 sets (seed 4):
the split entry points, for ncu.   python tools/split_prof_run.py [N]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from gen.inputs import config3_params
from paper_2404_06452_b200 import paam
gp = config3_params()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
raw = paam.Raw(paam.PaamGenParams.from_buffer_copy(bytes(gp)), 4, 0, n)
sets = paam.Sets(raw)
dev = torch.device("cuda")
w = torch.empty(raw.c.n_chains, dtype=torch.int64, device=dev)
s = torch.empty(n, dtype=torch.uint8, device=dev)
b = torch.zeros(2 * gp.n_bins, dtype=torch.int64, device=dev)
sets.analyze(w, s, b)
torch.cuda.synchronize()
print("ok", n)
