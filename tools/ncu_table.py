"""Summarise an `ncu --csv --metrics ...` log: one row per kernel launch."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idi = hdr.index("ID")
by = {}
order = []
for r in rows[1:]:
    key = (r[idi], r[ki])
    if key not in by:
        by[key] = {}
        order.append(key)
    by[key][r[mi]] = (r[vi], r[ui])
short = {"gpu__time_duration.sum": "time", "smsp__inst_executed.sum": "inst",
         "dram__bytes_read.sum": "dram_rd", "dram__bytes_write.sum": "dram_wr",
         "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
         "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
         "launch__registers_per_thread": "regs", "launch__grid_size": "grid"}
print(" | ".join(["kernel"] + list(short.values())))
for key in order:
    name = key[1]
    nm = name.split("(")[0].replace("void fllf::(anonymous namespace)::", "")
    if "<" in name:
        nm = name[name.index("k_"):name.index(">") + 1] if "k_" in name else nm
    vals = [f"{by[key].get(m, ('', ''))[0]} {by[key].get(m, ('', ''))[1]}".strip() for m in short]
    print(" | ".join([nm[:40]] + vals))
