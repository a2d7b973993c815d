"""Summarize an `ncu --metrics gpu__time_duration.sum --csv` launch list (dev aid)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
mi = hdr.index("Metric Name")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot, cnt = {}, {}
for r in rows[h + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":  # other metrics (grid size) are not times
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot[name] = tot.get(name, 0.0) + v
    cnt[name] = cnt.get(name, 0) + 1
T = sum(tot.values())
print(f"launch list: {sum(cnt.values())} launches, {T/1e3:.1f} ms device time (cold-cache, serialised by ncu)")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:70]:70s} n={cnt[k]:6d} total={tot[k]/1e3:9.3f} ms share={tot[k]/T:6.2%} avg={tot[k]/cnt[k]:9.2f} us")
