"""Hottest SASS instructions (warp-stall samples) of one kernel in an ncu report.

    python tools/ncu_hot.py REP.ncu-rep KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "--kernel-name",
                      "regex:" + kre, "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
data = [r for r in rows[rows.index(h) + 1:] if len(r) >= len(h) - 1 and r[0].startswith("0x")]
si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[si] or 0) for r in data)
print(rows[0][1][:120])
print(f"total stall samples {tot:.0f}, instructions {sum(float(r[ii] or 0) for r in data):.0f}")
for n, r in enumerate(data):
    r.append(n)
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:top]:
    reasons = sorted(((float(r[i] or 0), c[6:]) for i, c in stall_cols), reverse=True)[:2]
    print(f"{float(r[si]):6.0f} {100 * float(r[si]) / tot:5.1f}%  #{r[-1]:5d} {r[1].strip()[:60]:60s} exec {r[ii]:>8s}  {reasons}")
