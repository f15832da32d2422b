"""Where the time of an e2e step with device generation goes (host wall clock, synchronised parts)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from gen.inputs import config3_params
from paper_2404_06452_b200 import paam

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
gp = config3_params()
pp = paam.PaamGenParams.from_buffer_copy(bytes(gp))
st = torch.cuda.Stream()
raw = paam.Raw(pp, 4, 0, n, stream=st)
sets = paam.Sets(raw, stream=st)
sched = torch.empty(n, dtype=torch.uint8, device="cuda")
bins = torch.zeros(2 * gp.n_bins, dtype=torch.int64, device="cuda")
for it in range(5):
    t0 = time.perf_counter()
    raw.regenerate(pp, 4, 0, n, stream=st)
    st.synchronize(); t1 = time.perf_counter()
    sets.pack_analyze(raw, None, sched, bins, stream=st)
    st.synchronize(); t2 = time.perf_counter()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"generate {1e3*(t1-t0):.1f} ms  pack_analyze {1e3*(t2-t1):.1f} ms  sync {1e3*(t3-t2):.1f} ms", flush=True)
