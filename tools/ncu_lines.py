"""Stall samples per CUDA source line from an ncu `--page source --print-source cuda,sass` CSV
(experiments only): python tools/ncu_lines.py x_cudasass.csv[.gz] [top]"""
import collections
import csv
import gzip
import sys

f = sys.argv[1]
rows = list(csv.reader(gzip.open(f, "rt") if f.endswith(".gz") else open(f)))
out = collections.Counter()
reasons = collections.defaultdict(collections.Counter)
src = {}
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == "File Path":
        path = r[1].split("/")[-1]
        h = rows[i + 2]
        il, iall = h.index("Line No"), h.index("Warp Stall Sampling (All Samples)")
        st = {x: k for k, x in enumerate(h) if x.startswith("stall_")}
        i += 3
        while i < len(rows) and rows[i] and rows[i][0] != "File Path":
            r = rows[i]
            if r[il].strip().isdigit():
                key = (path, int(r[il]))
                src[key] = r[1].strip()[:80]
                try:
                    out[key] += int(r[iall] or 0)
                    for name, k in st.items():
                        reasons[key][name[6:]] += int(r[k] or 0)
                except (ValueError, IndexError):
                    pass
            i += 1
    else:
        i += 1
tot = sum(out.values()) or 1
for key, v in out.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    top = ", ".join(f"{k} {c / max(1, v):.2f}" for k, c in reasons[key].most_common(3) if c)
    print(f"{key[0]}:{key[1]:5d} {v / tot:6.3f}  [{top}]  {src[key]}")
