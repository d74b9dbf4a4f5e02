"""Config 5 throughput with the 64 frames split over S plans on S concurrent
streams (S = 1, 2, 4): do the kernels of one sub-batch fill the tails /
waves of the other's?  Device-timed with CUDA events (L2 flushed before each
step), interleaved repeats.  usage: python tools/stream_split_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_04681_b200 import fllf as F  # noqa: E402
from paper_2206_04681_b200 import synth  # noqa: E402

c = synth.CONFIGS[5]
H, W, L, K = c["H"], c["W"], c["levels"], c["K"]
N = 64
imgs = torch.from_numpy(synth.config5_frames(N)).cuda()
out = torch.empty_like(imgs)
flush_buf = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda")
main = torch.cuda.current_stream()


def setup(S):
    n = N // S
    plans = [F.Plan(H, W, L, K, c["T"], c["sigma_r"], c["m"], batch=n) for _ in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    return n, plans, streams


def step(S, n, plans, streams):
    ev = torch.cuda.Event()
    ev.record(main)
    for i in range(S):
        streams[i].wait_event(ev)
        plans[i].filter(imgs[i * n:(i + 1) * n], out[i * n:(i + 1) * n], streams[i])
    for s in streams:
        e = torch.cuda.Event()
        e.record(s)
        main.wait_event(e)


def timeit(S, cfg, steps=20):
    tot = 0.0
    for _ in range(steps):
        flush_buf.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        step(S, *cfg)
        b.record(main)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / steps


cfgs = {S: setup(S) for S in (1, 2, 4)}
for S, cfg in cfgs.items():
    for _ in range(3):
        step(S, *cfg)
torch.cuda.synchronize()
res = {S: [] for S in cfgs}
for rep in range(4):
    for S, cfg in cfgs.items():
        res[S].append(timeit(S, cfg))
for S, v in res.items():
    ms = sorted(v)
    print(f"S={S}: ms/step {['%.3f' % x for x in v]}  best {ms[0]:.3f}  -> {N * H * W / 1e6 / (ms[0] / 1e3):.0f} MP/s")
ref = out.clone()
step(1, *cfgs[1])
torch.cuda.synchronize()
a = out.clone()
step(4, *cfgs[4])
torch.cuda.synchronize()
print("S=4 vs S=1 max|diff|", float((out - a).abs().max()))
