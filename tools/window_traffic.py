"""DRAM traffic of the constant-row window launches from a SINGLE-PASS ncu run (experiments /
evidence). `ncu --set full` replays a kernel ~40 times and saves / restores the device buffers it
writes between passes, which shows up as DRAM traffic of the profiled launch; two metrics fit in
one pass, so no replay and no restore:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --cache-control none --csv --log-file gpurun_out/win_traffic.csv \
        -k regex:sweep_kernel_rc -s 60 -c 200 python tools/time_c4.py C4aamp C4acamp
    python tools/window_traffic.py gpurun_out/win_traffic.csv <tag>

Writes profiles/<tag>_window_traffic.txt and sets dram_bytes_per_launch in
profiles/ncu_summary.json to the mean read+write bytes per window launch."""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rows = list(csv.reader(open(sys.argv[1])))
tag = sys.argv[2]
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, ui, vi, idi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                       h.index("Metric Value"), h.index("ID"))
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}
per = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(r[idi], {"kernel": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", "")) * mult.get(r[ui], 1)
out = [f"# single-pass ncu of {len(per)} consecutive window launches (cache control none)"]
by = {}
for d in per.values():
    b = by.setdefault(d["kernel"][:80], {"n": 0, "rd": 0.0, "wr": 0.0, "us": 0.0})
    b["n"] += 1
    b["rd"] += d.get("dram__bytes_read.sum", 0.0)
    b["wr"] += d.get("dram__bytes_write.sum", 0.0)
    b["us"] += d.get("gpu__time_duration.sum", 0.0)
tot_n = sum(b["n"] for b in by.values())
tot_b = sum(b["rd"] + b["wr"] for b in by.values())
for k, b in by.items():
    out.append(f"{k}: {b['n']} launches, mean read {b['rd'] / b['n'] / 1e6:.2f} MB, "
               f"write {b['wr'] / b['n'] / 1e6:.2f} MB, duration {b['us'] / b['n']:.1f} us")
out.append(f"mean read+write per window launch: {tot_b / tot_n / 1e6:.2f} MB")
(ROOT / "profiles" / f"{tag}_window_traffic.txt").write_text("\n".join(out) + "\n")
print("\n".join(out))
f = ROOT / "profiles" / "ncu_summary.json"
js = json.loads(f.read_text()) if f.exists() else {}
js["dram_bytes_per_launch"] = tot_b / tot_n
js["dram_bytes_per_launch_source"] = (f"profiles/{tag}_window_traffic.txt: single-pass ncu, mean over {tot_n} "
                                      "window launches (--set full replays restore buffers between passes and "
                                      "inflate this metric)")
f.write_text(json.dumps(js, indent=1))
