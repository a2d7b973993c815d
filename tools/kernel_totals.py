"""Dev aid: total / mean device time per kernel name from an ncu launch list."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]; ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
L = {}
for r in rows[h + 1:]:
    if len(r) <= vi: continue
    d = L.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "").replace("shl::<unnamed>::", "")})
    d[r[mi]] = r[vi]
agg = defaultdict(list)
for d in L.values():
    key = d["name"][:50] + " g=" + d.get("launch__grid_size", "")
    agg[key].append(float(d["gpu__time_duration.sum"].replace(",", "")) / 1000)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{k:62s} n={len(v):4d} mean={sum(v)/len(v):8.1f} us total={sum(v)/1000:7.2f} ms {100*sum(v)/tot:5.1f}%")
print(f"all kernels {tot/1000:.2f} ms over {sum(len(v) for v in agg.values())} launches")
