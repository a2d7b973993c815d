"""Write profiles/ncu_summary.json (per-node DRAM bytes per kernel, read by
bench.py for roofline.traffic) from ncu --set full reports.
    python tools/ncu_json.py NODES "source text" rep1.ncu-rep [rep2 ...]"""
import csv, io, json, subprocess, sys
from collections import defaultdict

nodes, source, reps = int(sys.argv[1]), sys.argv[2], sys.argv[3:]
acc = defaultdict(list)
for rep in reps:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1]
        base = name.split("<")[0]
        g = lambda k: float(r[h.index(k)].replace(",", "")) * scale[units[h.index(k)]]
        acc[base].append((name, g("dram__bytes_read.sum"), g("dram__bytes_write.sum"), g("gpu__time_duration.sum"),
                          h, r))
out = {"source": source, "note": "per-node DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) / active "
       "level-0 nodes, longest captured launch of each kernel (ncu --set full, cold cache; coarse-level instances are smaller); bench.py scales by its "
       "own node count", "nodes": nodes, "kernels": {}}
for base, v in acc.items():
    name, rd, wr, us, h, r = max(v, key=lambda e: e[3])  # the longest captured launch (level 0)
    out["kernels"][base] = {"instance": name, "launches_captured": len(v), "dram_read_mb": round(rd / 1e6, 3),
                            "dram_write_mb": round(wr / 1e6, 3), "per_node_bytes": round((rd + wr) / nodes, 1),
                            "duration_us": round(us, 2)}
json.dump(out, open("profiles/ncu_summary.json", "w"), indent=1)
print(json.dumps(out, indent=1))
