"""Time fllf_filter (graph + PDL, unprofiled) for ad-hoc shapes: prints us/step.
    python tools/time_filter.py H W levels K [frames]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2206_04681_b200 import fllf as F  # noqa: E402
from paper_2206_04681_b200 import synth  # noqa: E402

H, W, L, K = map(int, sys.argv[1:5])
B = int(sys.argv[5]) if len(sys.argv) > 5 else 1
x = torch.from_numpy(synth.uniform_image(H, W, seed=1)).cuda().expand(B, H, W).contiguous()
o = torch.empty_like(x)
flush = torch.empty(64 << 20, device="cuda")
with F.Plan(H, W, L, K, 510.0, 30.0, 3.0, batch=B) as p:
    for _ in range(5):
        p.filter(x, o)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
    for a, b in ev:
        flush.zero_()
        a.record()
        p.filter(x, o)
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    print(f"{H}x{W} L{L} K{K} B{B}: median {t[len(t)//2]*1e3:.1f} us  min {t[0]*1e3:.1f} us")
