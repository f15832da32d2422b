"""Per-CUDA-source-line instruction and stall totals of one kernel in an .ncu-rep:
python tools/ncu_lines.py rep kernel_regex [top]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
key = 0 if len(sys.argv) > 4 and sys.argv[4] == "inst" else 1  # sort by instructions or by stall samples
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0, ""])
cur = "?"
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    inst = int(r[hdr.index("Instructions Executed")] or 0)
    st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    a = agg[(cur, ln)]
    a[0] += inst; a[1] += st
    if not a[2]:
        a[2] = r[1][:90]
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total inst {tot_i}  samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
    print(f"{k[0]}:{k[1]:4d} inst {100*v[0]/tot_i:5.1f}%  stall {100*v[1]/tot_s:5.1f}%  {v[2].strip()}")
