"""Dev aid: per-kernel device time of one PCG iteration from an ncu launch list."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]; ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
L, order = {}, []
for r in rows[h + 1:]:
    if len(r) <= vi: continue
    if r[ii] not in L: order.append(r[ii])
    d = L.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "").replace("shl::<unnamed>::", "")})
    d[r[mi]] = r[vi]
seq = [(L[i]["name"][:44], L[i].get("launch__grid_size", ""), float(L[i]["gpu__time_duration.sum"].replace(",", "")) / 1000) for i in order]
ch = [i for i, s in enumerate(seq) if "chom" in s[0]]
ups = [i for i in range(ch[-2] if len(ch) > 1 else 0, ch[-1]) if "update_kernel" in seq[i][0]]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 5
a, b = ups[k], ups[k + 1]
tot = 0
for s in seq[a:b]:
    print(f"{s[0]:46s} grid={s[1]:>6s} {s[2]:8.1f} us"); tot += s[2]
print(f"iteration total {tot:.1f} us over {b-a} launches")
