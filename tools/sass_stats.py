"""Per-kernel SASS statistics from `cuobjdump -sass` output (experiments only):
    python tools/sass_stats.py file.sass [name-substring ...]
Counts DFMA / DADD / DMUL, how many carry a .reuse flag, VIMNMX3 / IMNMX / LDS / BAR."""
import re
import sys
from collections import Counter

text = open(sys.argv[1]).read()
pats = sys.argv[2:] or ["sweep_kernel"]
funcs = re.split(r"\n\s+Function : ", text)
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    if not all(p in name for p in pats):
        continue
    ins = re.findall(r"/\*[0-9a-f]{4}\*/\s+([^;]*);", f)
    c = Counter()
    for i in ins:
        op = i.split()[0] if not i.startswith("@") else i.split()[1]
        base = op.split(".")[0]
        c[base] += 1
        if base in ("DFMA", "DADD", "DMUL") and ".reuse" in i:
            c[base + ".reuse"] += 1
            c[base + ".reuse_ops"] += i.count(".reuse")
    print(name[:110])
    print("  ", {k: c[k] for k in ("DFMA", "DFMA.reuse", "DFMA.reuse_ops", "DADD", "DMUL", "VIMNMX3",
                                   "VIMNMX", "IMNMX", "LDS", "BAR", "BRA") if c[k]}, "total", len(ins))
