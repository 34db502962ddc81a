"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

    python tools/ncu_summary.py <tag> [--launches gpurun_out/launches.csv] [--rep gpurun_out/prof.ncu-rep]

Writes profiles/<tag>_launches.txt (per-kernel share of the launch list) and
profiles/<tag>_ncu.txt + profiles/ncu_summary.json (key counters of each profiled kernel:
FP64 pipe, issue, occupancy, stall reasons, DRAM traffic per launch, shared-memory wavefronts).
"""
import argparse
import csv
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "lts__t_bytes.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
    "l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum",
    "smsp__inst_executed_op_global_atom.sum",
]


def launches(path: Path, tag: str):
    rows = list(csv.reader(path.open()))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = {}, {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki]
        tot[name] = tot.get(name, 0.0) + float(r[vi].replace(",", ""))
        cnt[name] = cnt.get(name, 0) + 1
    s = sum(tot.values())
    out = [f"# ncu launch list ({path.name}): gpu__time_duration.sum per kernel, cold-cache serialised",
           f"# total {s / 1e6:.3f} ms over {sum(cnt.values())} launches", ""]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{v / 1e6:11.3f} ms {100 * v / s:6.2f}%  x{cnt[k]:<3d} {k[:110]}")
    (ROOT / "profiles" / f"{tag}_launches.txt").write_text("\n".join(out) + "\n")
    print("\n".join(out))


def _rows(rep: Path):
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    return rows[0], rows[1], rows[2:]


def full(reps, tag: str):
    summary = {}
    lines = [f"# ncu --set full summary ({', '.join(r.name for r in reps)})"]
    for h, units, r in ((h, u, r) for rep in reps for h, u, rs in [_rows(rep)] for r in rs):
        name = r[h.index("Kernel Name")]
        d = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        stalls = {}
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(r[i])
                except ValueError:
                    pass
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:10])
        summary.setdefault(name, d)
        lines.append(f"\n## {name}")
        for k, v in d.items():
            lines.append(f"  {k}: {v}")
    (ROOT / "profiles" / f"{tag}_ncu.txt").write_text("\n".join(lines) + "\n")
    # per-launch DRAM traffic of the dominant kernel(s) for bench.py's roofline.traffic
    traffic = {}
    for name, d in summary.items():
        try:
            def nbytes(text):  # "31.5 Mbyte" -> bytes (each metric carries its own unit)
                val, unit = text.split()[:2]
                return float(val) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            traffic[name] = nbytes(d["dram__bytes_read.sum"]) + nbytes(d["dram__bytes_write.sum"])
        except (KeyError, ValueError, IndexError):
            pass
    js = {"tag": tag, "kernels": summary, "dram_bytes_per_launch_by_kernel": traffic,
          "dram_bytes_per_launch": max(traffic.values()) if traffic else None}
    (ROOT / "profiles" / "ncu_summary.json").write_text(json.dumps(js, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches", default=str(ROOT / "gpurun_out" / "launches.csv"))
    ap.add_argument("--rep", action="append", default=None, help="repeatable")
    a = ap.parse_args()
    if Path(a.launches).exists():
        launches(Path(a.launches), a.tag)
    reps = [Path(r) for r in (a.rep or [str(ROOT / "gpurun_out" / "prof.ncu-rep")]) if Path(r).exists()]
    if reps:
        full(reps, a.tag)
