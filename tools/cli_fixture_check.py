"""Runs the CLI on the three acceptance fixtures the way the reference's criterion 11 does and
prints exit codes and stderr (experiments / debugging)."""
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
g = np.load(ROOT / "tests" / "golden" / "fixtures.npz")
out = Path("/tmp/fx")
out.mkdir(exist_ok=True)
for name, flags in (("euclidean", "--distance euclidean"), ("pnorm", "--distance pnorm --p 3"),
                    ("znorm", "--distance znorm")):
    f = out / f"fixture_{name}.csv"
    f.write_text("value\n" + "\n".join(repr(float(x)) for x in g[f"{name}_t"]) + "\n")
    for extra in ("", " --engine oracle"):
        cmd = f"{ROOT}/paper_1901_05708_b200/bin/mprof compute --input {f} --m 50 {flags}{extra}"
        r = subprocess.run(cmd, shell=True, capture_output=True, text=True)
        print(name, extra, "exit", r.returncode, "stderr:", r.stderr.strip()[:300], "lines", r.stdout.count("\n"))
