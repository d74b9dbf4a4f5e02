"""Small fixed workload for ncu captures: N filter calls of one BASELINE config.

    python tools/ncu_target.py [--workload config2|config5|config3|config4] [--iters 2]
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
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--frames", type=int, default=16)
    ap.add_argument("--maps", action="store_true", help="config 4: build once, then one MAPS apply")
    ap.add_argument("--fused-levels", type=int, default=-1,
                    help="design F on levels 1..N (0: AUTO for this batch; -1: as the 64-frame bench picks)")
    a = ap.parse_args()
    cfg = int(a.workload[-1])
    c = synth.CONFIGS[cfg]
    if cfg == 5:
        x = synth.config5_frames(a.frames)
    elif cfg in (3, 4):
        x = synth.config2_image(seed=4000, H=c["H"], W=c["W"])[None]
    else:
        x = synth.config2_image()[None] if cfg == 2 else synth.config1_image()[None]
    d_in = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    d_out = torch.empty_like(d_in)
    sig = c.get("sigma_r", 30.0)
    m = c.get("m", 2.0)
    with F.Plan(c["H"], c["W"], c["levels"], c["K"], c["T"], sig, m, batch=d_in.shape[0]) as p:
        if a.maps:
            s_map, m_map = (torch.from_numpy(v).cuda() for v in synth.config4_maps(0, H=c["H"], W=c["W"]))
            p.build(d_in)
            for _ in range(a.iters):
                p.apply(d_out, mode=F.FLLF_MAPS, sigma_map=s_map, m_map=m_map)
            torch.cuda.synchronize()
            print("MAPS apply ok, out mean", float(d_out.mean()))
            return
        fl = a.fused_levels
        if fl < 0:  # the bench's choice at its own batch: F on the levels with >= 4 MP over 64 frames
            bench_batch = 64 if cfg == 5 else 1
            fl, h, w = 0, c["H"], c["W"]
            while fl < c["levels"] - 2:
                h, w = (h + 1) // 2, (w + 1) // 2
                if bench_batch * h * w < 4e6:
                    break
                fl += 1
            if fl == 0:
                F.fllf_plan_set_design(p.handle, F.FLLF_DESIGN_AB)
        if fl > 0:
            F.fllf_plan_set_fused_levels(p.handle, fl)
        for _ in range(a.iters):
            p.filter(d_in, d_out)
        torch.cuda.synchronize()
        print("launches per filter:", p.launches, "out mean", float(d_out.mean()))


if __name__ == "__main__":
    main()
