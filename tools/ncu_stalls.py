"""Warp stall breakdown (cycles per issued instruction by reason) of every kernel in an .ncu-rep:
python tools/ncu_stalls.py rep"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for v in rows[2:]:
    print("---", v[h.index("Kernel Name")][:60])
    for k, x in zip(h, v):
        if "smsp__average_warp" in k and "issue_stalled" in k and "ratio" in k:
            try:
                if float(x) > 0.1:
                    print("  %-28s %s" % (k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), x))
            except ValueError:
                pass
        if k in ("smsp__warps_eligible.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active"):
            print("  %-28s %s" % (k, x))
