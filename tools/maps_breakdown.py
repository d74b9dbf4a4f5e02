"""Per-kernel breakdown of one MAPS reapply at config 4 (4K, K = 12, 7 levels):
map-pyramid builds + MAPS applies, each bracketed by CUDA events (profiling
mode serialises the kernels).
    python tools/maps_breakdown.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2206_04681_b200 import fllf as F  # noqa: E402
from paper_2206_04681_b200 import synth  # noqa: E402


def main():
    c = synth.CONFIGS[4]
    H, W, levels, K = c["H"], c["W"], c["levels"], c["K"]
    img = torch.from_numpy(synth.config2_image(seed=4000, H=H, W=W)).cuda()
    s_map, m_map = (torch.from_numpy(m).cuda() for m in synth.config4_maps(0, H=H, W=W))
    out = torch.empty_like(img)
    with F.Plan(H, W, levels, K, c["T"], 30.0, 1.0) as p:
        p.build(img)
        F.fllf_plan_set_profiling(p.handle, True)
        acc = {}
        n = 20
        for _ in range(n):
            p.apply(out, mode=F.FLLF_MAPS, sigma_map=s_map, m_map=m_map)
            for kind, lev, ms in F.fllf_plan_kernel_times(p.handle):
                acc.setdefault((kind, lev), []).append(ms)
        torch.cuda.synchronize()
        tot = sum(sum(v) for v in acc.values()) / n
        for (kind, lev), v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
            print(f"{kind:9s} l={lev}  {sum(v) / len(v) * 1e3:8.2f} us  {sum(v) / n / tot:6.1%}")
        print(f"sum {tot * 1e3:.1f} us per reapply (serialised)")


if __name__ == "__main__":
    main()
