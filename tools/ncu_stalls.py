"""Stall reasons per SASS address range of one kernel in an ncu --set full report (diagnostics).

    python tools/ncu_stalls.py <report.ncu-rep> a:b[:name] [a:b[:name] ...]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, body = rows[1], rows[2:]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in reasons}
tot = sum(int(x[h.index("Warp Stall Sampling (All Samples)")]) for x in body)
for spec in sys.argv[2:]:
    parts = spec.split(":")
    a, b = int(parts[0]), int(parts[1])
    name = parts[2] if len(parts) > 2 else spec
    sums = {c: sum(int(x[idx[c]] or 0) for x in body[a:b]) for c in reasons}
    t = sum(sums.values())
    top = sorted(sums.items(), key=lambda kv: -kv[1])[:6]
    print(f"{name:14s} {100 * t / tot:5.1f}%  " + "  ".join(f"{k[6:]} {100 * v / max(t, 1):.0f}%" for k, v in top))
