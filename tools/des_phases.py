"""Per-phase instruction / stall shares of simulate_kernel from an .ncu-rep (source page), the phases
found from the marker comments of the current csrc/simulate.cu.   python tools/des_phases.py rep"""
import csv, io, os, re, subprocess, sys
from collections import defaultdict
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = open(os.path.join(ROOT, "paper_2404_06452_b200", "csrc", "simulate.cu")).read().splitlines()
marks = [("fnv_time(", "digest fns"), ("struct Ctx", "ctx/ev/flush"), ("bool begin_segment", "begin_seg"),
         ("bool advance_segment", "advance_seg"), ("__global__", "setup"), ("settle time t", "(1) units"),
         ("// (2) executors", "(2) execs"), ("// (3) comm arrivals", "(3)(4)+vote"),
         ("must_flush()) C.flush(lane);\n", None), ("// (5) executor choice", "(5) exec choice"),
         ("// (6) core dispatch", "(6) core"), ("// (7) unit dispatch", "(7) units"),
         ("advance time =", "advance t"), ("---- outputs", "outputs"), ("#ifndef PAAM_WARP_EMU\nint launch", "end")]
starts = []
for i, l in enumerate(src, 1):
    if i < 40:  # the header comment names the phases too
        continue
    for m, name in marks:
        if name and m.split("\n")[0] in l and not any(s[1] == name for s in starts):
            starts.append((i, name))
starts.sort()
def phase(ln):
    name = "misc"
    for s, n in starts:
        if ln >= s:
            name = n
    return name
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass,cuda", "-k", "regex:simulate"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0]); cur = "?"; hdr = None; tot = [0, 0]
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    try: ln = int(r[0])
    except ValueError: continue
    i = int(r[hdr.index("Instructions Executed")] or 0); s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    tot[0] += i; tot[1] += s
    name = phase(ln) if cur == "simulate.cu" else cur
    agg[name][0] += i; agg[name][1] += s
print(f"total warp instructions {tot[0]}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:28s} inst {100 * v[0] / tot[0]:5.1f}%  stall {100 * v[1] / tot[1]:5.1f}%")
