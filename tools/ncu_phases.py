"""Aggregate per-source-line instruction counts / stall samples of one kernel by code phase, where a
phase starts at every comment line containing '----' in the kernel's source file.
python tools/ncu_phases.py rep kernel_regex source_file"""
import csv, io, subprocess, sys
from collections import defaultdict
rep, kre, src = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
lines = open(src).read().splitlines()
marks = [(i + 1, l.strip()[:70]) for i, l in enumerate(lines) if "----" in l and l.strip().startswith("//")]
def phase(ln):
    name = "prologue"
    for m, t in marks:
        if m <= ln: name = f"{m}: {t}"
    return name
agg = defaultdict(lambda: [0, 0]); cur = None; hdr = None
base = src.split("/")[-1]
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    try: ln = int(r[0])
    except ValueError: continue
    key = phase(ln) if cur == base else f"(inlined {cur})"
    agg[key][0] += int(r[hdr.index("Instructions Executed")] or 0)
    agg[key][1] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
ti = sum(v[0] for v in agg.values()) or 1; ts = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: kv[0]):
    print(f"inst {100*v[0]/ti:5.1f}%  stall {100*v[1]/ts:5.1f}%  {k}")
