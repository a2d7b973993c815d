"""dev aid: per-phase timeline of CTA 0 from a SHL_BRICK_TRACE run (tools/brick_trace.sh)."""
import re, sys
recs = []
for l in open(sys.argv[1]):
    m = re.match(r'(\w+) cta (\d) (\w) line (\d+) t (\d+)', l)
    if m:
        recs.append((m.group(1), int(m.group(2)), m.group(3), int(m.group(4)), int(m.group(5))))
kern = sys.argv[2] if len(sys.argv) > 2 else 'apply'
lines = sorted({r[3] for r in recs})
cur = sorted([r for r in recs if r[0] == kern and r[1] == 0], key=lambda r: r[4])
groups, g = [], []
for r in cur:
    if g and r[4] - g[-1][4] > 50000:
        groups.append(g)
        g = []
    g.append(r)
groups.append(g)
G = groups[-1]
t0 = G[0][4]
for r in G[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(kern, r[2], r[3], f"{(r[4] - t0) / 1000:8.2f} us")
