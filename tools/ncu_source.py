"""Per-region stall attribution from an ncu source page (SASS) CSV:
    ncu -i rep --page source --csv --print-source sass > x.csv; python tools/ncu_source.py x.csv
Prints the hottest instruction windows (by stall samples) with their stall-reason mix."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
ri = {r: h.index(r) for r in reasons}
tot = Counter()
total = 0
ins = []
for r in data:
    try:
        s = int(r[iall])
    except ValueError:
        continue
    total += s
    c = {k: int(r[i] or 0) for k, i in ri.items()}
    tot.update(c)
    ins.append((r[ia], r[isrc].strip(), s, c))
print("total samples", total)
print("by reason:", {k: round(v / total, 3) for k, v in tot.most_common(12)})
W = int(sys.argv[2]) if len(sys.argv) > 2 else 64
# windows of W instructions
best = []
for a in range(0, len(ins), W // 2):
    w = ins[a:a + W]
    s = sum(x[2] for x in w)
    best.append((s, a))
best.sort(reverse=True)
for s, a in best[:6]:
    w = ins[a:a + W]
    c = Counter()
    for x in w:
        c.update(x[3])
    print(f"\nwindow {a}..{a + W} ({w[0][0][-5:]}): {s / total:.3f} of samples;",
          {k[6:]: round(v / max(1, s), 2) for k, v in c.most_common(6)})
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[3]), int(sys.argv[4])
    for x in ins[lo:hi]:
        top = sorted(x[3].items(), key=lambda kv: -kv[1])[:3]
        print(f"{x[0][-5:]} {x[2]:7d} {x[1][:60]:60s} {[(k[6:], v) for k, v in top if v]}")
