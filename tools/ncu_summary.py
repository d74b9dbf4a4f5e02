"""Summarise an ncu report (--set full) into markdown + roofline traffic json.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_full.md [workload [levels [frames]]]

With `levels`, the launches are taken as one filter sequence (build0,
build 1..levels-2, apply levels-2..1, apply0) and their DRAM read+write bytes
PER FRAME (the capture's bytes / `frames`, the batch the capture ran) are
merged into profiles/roofline_traffic.json under "<workload>:<kind>:<level>";
bench.py multiplies by its own batch for the roofline `traffic` field.
"""
import csv
import re
import io
import json
import os
import subprocess
import sys

rep, out_md = sys.argv[1], sys.argv[2]
workload = sys.argv[3] if len(sys.argv) > 3 else "config2"
# an .ncu-rep, or its raw page already exported (`ncu -i REP --page raw --csv`)
raw = open(rep).read() if rep.endswith(".csv") else \
    subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]


def g(r, k):
    return r[hdr.index(k)] if k in hdr else ""


stall_cols = [i for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
lines = ["| # | kernel | time (us) | DRAM read (MB) | DRAM write (MB) | regs | occupancy % | issue active % | FMA pipe % | L1 % | top stalls (cycles/issue) |",
         "|---|---|---|---|---|---|---|---|---|---|---|"]
traffic = {}
seen = {}
for n, r in enumerate(data):
    name = g(r, "Kernel Name")
    short = name[name.find("k_"):name.find("(")] if "k_" in name else name[:40]
    t_us = float(g(r, "gpu__time_duration.sum") or 0)
    tu = units[hdr.index("gpu__time_duration.sum")]
    if tu == "ns":
        t_us /= 1e3
    elif tu == "ms":
        t_us *= 1e3

    def mb(k):
        v = float(g(r, k) or 0)
        u = units[hdr.index(k)] if k in hdr else "byte"
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
        return v * scale

    rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
    st = sorted(((float(r[i] or 0), hdr[i].replace("smsp__average_warps_issue_stalled_", "")
                  .replace("_per_issue_active.ratio", "")) for i in stall_cols), reverse=True)[:3]
    lines.append(f"| {n} | `{short}` | {t_us:.2f} | {rd:.2f} | {wr:.2f} | {g(r, 'launch__registers_per_thread')} | "
                 f"{float(g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                 f"{float(g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                 f"{float(g(r, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                 f"{float(g(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                 + ", ".join(f"{nm} {v:.2f}" for v, nm in st) + " |")
    seen.setdefault(short, []).append((rd + wr) * 1e6)
# roofline traffic per (kind, level) for the sequence order build0..build(l), apply(l)..apply0
md = [f"# ncu --set full summary: `{os.path.basename(rep)}` ({workload})", "",
      "Per launch, cold caches (ncu replays each kernel with caches flushed), --clock-control none.", ""] + lines
open(out_md, "w").write("\n".join(md) + "\n")
print("\n".join(md))
if len(sys.argv) > 4:
    # argv[4]: the launch sequence of one filter, comma-separated kind+level
    # (e.g. build0,fuse1,fuse2,build3,build4,apply4,apply3,collapse2,collapse1,apply0)
    # or a level count for the design-AB order
    spec = sys.argv[4]
    if spec.isdigit():
        levels = int(spec)
        order = [("build0", 0)] + [("build", l) for l in range(1, levels - 1)] + \
                [("apply", l) for l in range(levels - 2, 0, -1)] + [("apply0", 0)]
    else:
        order = []
        for item in spec.split(","):
            m = re.match(r"([a-z]+?)(\d+)$", item)
            kind, lev = m.group(1), int(m.group(2))
            order.append((kind if not (kind == "build" and lev == 0) else "build0", lev))
    rows_bytes = []
    for r in data:
        def mbv(k):
            v = float(g(r, k) or 0)
            u = units[hdr.index(k)] if k in hdr else "byte"
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        rows_bytes.append(mbv("dram__bytes_read.sum") + mbv("dram__bytes_write.sum"))
    if len(rows_bytes) >= len(order):
        tp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                          "roofline_traffic.json")
        tj = json.load(open(tp)) if os.path.exists(tp) else {}
        frames = int(sys.argv[5]) if len(sys.argv) > 5 else 1
        for (kind, lev), b in zip(order, rows_bytes[:len(order)]):
            tj[f"{workload}:{kind}:{lev}"] = round(b / frames)
        json.dump(tj, open(tp, "w"), indent=1, sort_keys=True)
        print("traffic ->", tp)
        if len(sys.argv) > 6:  # argv[6]: pixels per frame -> DRAM bytes per pixel of the whole sequence
            px = float(sys.argv[6])
            tot = sum(rows_bytes[:len(order)]) / frames
            with open(out_md, "a") as f:
                f.write(f"\nWhole filter sequence: DRAM {tot / 1e6:.1f} MB per frame = {tot / px:.1f} B per level-0 "
                        f"pixel (read + write, cold caches).\n")
