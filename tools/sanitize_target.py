"""Small cases for compute-sanitizer (memcheck / racecheck / initcheck): config 1,
odd sizes with unaligned pitch, MAPS mode, order ranges, batch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2206_04681_b200 import fllf as F  # noqa: E402
from paper_2206_04681_b200 import synth  # noqa: E402


def run(H, W, levels, K, **kw):
    B = kw.pop("batch", 1)
    x = torch.from_numpy(np.stack([synth.uniform_image(H, W, seed=s) for s in range(B)])).cuda()
    o = torch.empty_like(x)
    with F.Plan(H, W, levels, K, 510.0, 30.0, 2.0, batch=B, **kw) as p:
        p.filter(x, o)
        s = torch.rand((H, W), device="cuda") * 50 + 10
        m = torch.rand((H, W), device="cuda") * 3 + 0.5
        p.apply(o, mode=F.FLLF_MAPS, sigma_map=s, m_map=m)
        torch.cuda.synchronize()
    assert torch.isfinite(o).all()


run(256, 256, 4, 4)
run(37, 23, 3, 5)
run(121, 300, 6, 16)
run(259, 130, 7, 1)
run(64, 33, 2, 10, k_begin=3, k_end=8, include_base=False)
run(40, 52, 4, 7, batch=3)
print("sanitize target done")

# NEXT-3 colour pipeline and NEXT-2 naive LLF
rgb = torch.rand((3, 61, 90), device="cuda") * 255
out = torch.empty_like(rgb)
with F.Plan(61, 90, 4, 8, 510.0, 30.0, 1.0) as p:
    F.fllf_enhance_rgb(p.handle, rgb, out, 3, 0.5, 3.0, 120.0)
    img = rgb[0].contiguous()
    o2 = torch.empty_like(img)
    F.fllf_naive_llf(p.handle, img, o2, F.REMAP_EXACT)
    torch.cuda.synchronize()
assert torch.isfinite(out).all() and torch.isfinite(o2).all()
print("sanitize target (colour, naive) done")
