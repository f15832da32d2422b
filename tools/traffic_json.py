"""profiles/traffic.json from ncu --set full captures: per kernel DRAM bytes per set, issue-slot
utilisation and warp-instructions per set.   python tools/traffic_json.py out.json rep:kernel:sets ..."""
import csv, io, json, subprocess, sys
out = {"_about": "DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum), issue-slot utilisation "
                 "(smsp__issue_active.avg.pct_of_peak_sustained_active) and warp instructions "
                 "(smsp__inst_executed.sum) per set, from ncu --set full --clock-control none captures "
                 "(one launch each; sources listed per kernel)."}
for spec in sys.argv[2:]:
    rep, kern, sets = spec.split(":")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    for v in rows[2:]:
        if kern not in v[h.index("Kernel Name")]:
            continue
        g = lambda k: float(v[h.index(k)].replace(",", ""))
        # units: ncu reports each metric in the unit of its column (rows[1]); normalise to bytes
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = lambda k: g(k) * scale.get(rows[1][h.index(k)], 1)
        rd, wr, mul = b("dram__bytes_read.sum"), b("dram__bytes_write.sum"), 1
        inst = g("smsp__inst_executed.sum")
        n = int(sets)
        out[kern] = {"dram_read_bytes": rd * mul, "dram_write_bytes": wr * mul, "sets": n,
                     "dram_bytes_per_set": round((rd + wr) * mul / n, 1),
                     "issue_active_pct": round(g("smsp__issue_active.avg.pct_of_peak_sustained_active"), 2),
                     "warp_inst_per_set": round(inst / n, 1), "source": rep.split("/")[-1]}
        break
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1))
