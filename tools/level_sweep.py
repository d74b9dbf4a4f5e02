"""Marginal cost of pyramid levels: time fllf_filter on one workload shape with
levels = 2 .. L (CUDA graph replay, CUDA events, median of N).

    python tools/level_sweep.py [--workload config2] [--n 50]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2206_04681_b200 import fllf as F  # noqa: E402
from paper_2206_04681_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config2")
    ap.add_argument("--n", type=int, default=50)
    a = ap.parse_args()
    c = synth.CONFIGS[int(a.workload[-1])]
    x = torch.from_numpy(synth.config2_image(H=c["H"], W=c["W"])).cuda()
    y = torch.empty_like(x)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for L in range(2, c["levels"] + 1):
        with F.Plan(c["H"], c["W"], L, c["K"], c["T"], c.get("sigma_r", 30.0), c.get("m", 2.0)) as p:
            for _ in range(5):
                p.filter(x, y)
            ts = []
            for _ in range(a.n):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                p.filter(x, y)
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e) * 1e3)
            print(f"levels={L}: median {np.median(ts):.1f} us  min {np.min(ts):.1f} us  ({p.launches} launches)")


if __name__ == "__main__":
    main()
