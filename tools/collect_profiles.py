"""Copy one round's GPU artefacts from gpurun_out/ into profiles/ and write
the summaries (run here, after `gpurun -- 'bash tools/round_profiles.sh TAG;
bash tools/round_extra.sh TAG'`).

    python tools/collect_profiles.py TAG
"""
import csv
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def json_line(src, dst):
    """The bench's JSON line (drop library chatter such as NCCL's banner)."""
    lines = [ln for ln in open(src) if ln.lstrip().startswith("{")]
    if lines:
        open(dst, "w").write(lines[-1])


def kernels(src, dst):
    open(dst, "w").writelines(ln for ln in open(src) if ln.startswith("[bench]"))


def launch_summary(tag, step_us, seqlen, workload):
    rows = [r for r in csv.reader(open(os.path.join(PROF, f"{tag}_launches.csv"))) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ks = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:] if "k_" in r[ki]]
    seq = ks[-seqlen:]

    def short(n):
        m = re.search(r"(k_\w+)(<[^>]*>)?", n)
        return (m.group(1) + (m.group(2) or "")) if m else n

    tot = sum(v for _, v in seq) / 1e3
    md = [f"# ncu launch list (bench.py --steps 2 --warmup 1, {workload}), last filter sequence", "",
          "Cold-cache, serialised per-launch times (`--metrics gpu__time_duration.sum --clock-control none`). "
          "Compare shares, not absolutes.", "", "| # | kernel | us | share |", "|---|---|---|---|"]
    md += [f"| {i} | `{short(n)}` | {v / 1e3:.2f} | {v / 1e3 / tot:.1%} |" for i, (n, v) in enumerate(seq)]
    md += ["", f"Sum {tot:.1f} us serialised; the unprofiled bench step (PDL-overlapped graph) is {step_us:.1f} us."]
    open(os.path.join(PROF, f"{tag}_launches_summary.md"), "w").write("\n".join(md) + "\n")


# one filter sequence of the default bench (config 5, 64 frames: design F on
# levels 1-2, AB on 3-4) and of config 2 (design AB)
SEQ_C5 = "build0,fuse1,fuse2,build3,build4,apply4,apply3,collapse2,collapse1,apply0"
SEQ_C2 = "6"


def main():
    tag = sys.argv[1]
    src = lambda n: os.path.join(OUT, f"{tag}_{n}")  # noqa: E731
    dst = lambda n: os.path.join(PROF, f"{tag}_{n}")  # noqa: E731
    json_line(src("bench.json"), dst("bench_config5.json"))
    kernels(src("bench.err"), dst("bench_config5_kernels.txt"))
    for w in ("config2", "config4", "config3", "bands", "color"):
        if os.path.exists(src(f"bench_{w}.json")):
            json_line(src(f"bench_{w}.json"), dst(f"bench_{w}.json"))
    for w in ("config2", "config4"):
        if os.path.exists(src(f"bench_{w}.err")):
            kernels(src(f"bench_{w}.err"), dst(f"bench_{w}_kernels.txt"))
    for n in ("reference.json", "launches.csv", "clocks.csv", "gpu_tests.log", "c5_full_raw.csv", "c2_full_raw.csv"):
        if os.path.exists(src(n)):
            shutil.copy(src(n), dst(n))
    import json
    step_us = json.load(open(dst("bench_config5.json")))["ms_per_step"] * 1e3
    if os.path.exists(dst("launches.csv")):
        launch_summary(tag, step_us, len(SEQ_C5.split(",")), "config5")
    summ = os.path.join(ROOT, "tools", "ncu_summary.py")
    rep = lambda n: src(f"{n}.ncu-rep") if os.path.exists(src(f"{n}.ncu-rep")) else src(f"{n}_raw.csv")  # noqa: E731
    if os.path.exists(rep("c5_full")):  # 8 frames, the 64-frame bench's design
        subprocess.run([sys.executable, summ, rep("c5_full"), dst("ncu_full_config5.md"), "config5", SEQ_C5, "8",
                        str(1080 * 1920)],
                       check=True, stdout=subprocess.DEVNULL)
    if os.path.exists(rep("c2_full")):
        subprocess.run([sys.executable, summ, rep("c2_full"), dst("ncu_full_config2.md"), "config2", SEQ_C2, "1",
                        str(1080 * 1920)],
                       check=True, stdout=subprocess.DEVNULL)
    print("profiles written for", tag)


if __name__ == "__main__":
    main()
