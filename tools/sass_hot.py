"""Per-opcode and per-region stall breakdown of one kernel from an ncu source page
(dev aid): ncu -i rep --page source --csv --print-source sass -k regex:NAME > src.csv"""
import csv, sys
from collections import Counter, defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data, seen = [], set()
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    if r[0] in seen:
        break
    seen.add(r[0])
    data.append(r)
def num(x):
    try:
        return int(x)
    except ValueError:
        return 0
si, ii, src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(num(r[si]) for r in data)
by_op = defaultdict(Counter)
cnt = Counter()
for r in data:
    t = r[src].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    cnt[op] += num(r[ii])
    for h in reasons:
        by_op[op][h[6:]] += num(r[hdr.index(h)])
print(f"samples {tot}, warp-instructions {sum(cnt.values())}")
for op, c in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
    s = sum(c.values())
    print(f"{op:8s} inst {cnt[op]:>10d} samples {s:6d} ({s/tot:5.1%}): " +
          ", ".join(f"{k} {v/s:.0%}" for k, v in c.most_common(4) if v))
