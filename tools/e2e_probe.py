"""Streaming end-to-end probe (config 2): fllf_filter_host_frames over n
frames with / without the in-pipeline L2 flush, against the copy-only and
filter-only times of the same frames."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2206_04681_b200 import fllf as F  # noqa: E402
from paper_2206_04681_b200 import synth  # noqa: E402


def timed(fn, stream):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def main():
    n = 20
    img = synth.config2_image(seed=2000)
    H, W = img.shape
    h_in = torch.from_numpy(img).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    d_in = torch.from_numpy(img).cuda()
    d_out = torch.empty_like(d_in)
    fl = torch.empty(64 << 20, device="cuda")
    s = torch.cuda.current_stream()
    with F.Plan(H, W, 6, 8, 510.0, 30.0, 3.0) as p:
        F.fllf_filter_host_frames(p.handle, h_in, 0, h_out, 0, 2, s)
        torch.cuda.synchronize()
        for flush in (None, fl):
            F.fllf_plan_set_l2_flush(p.handle, flush)
            ms = timed(lambda: F.fllf_filter_host_frames(p.handle, h_in, 0, h_out, 0, n, s), s)
            print(f"host_frames flush={'on ' if flush is not None else 'off'}: {ms / n * 1e3:.1f} us/frame", flush=True)
        F.fllf_plan_set_l2_flush(p.handle, None)
        ms = timed(lambda: [p.filter(d_in, d_out, s) for _ in range(n)], s)
        print(f"filter only (device-resident):   {ms / n * 1e3:.1f} us/frame", flush=True)
        ms = timed(lambda: [F.fllf_filter_host(p.handle, h_in, h_out, s) for _ in range(n)], s)
        print(f"fllf_filter_host loop (serial):  {ms / n * 1e3:.1f} us/frame", flush=True)


if __name__ == "__main__":
    main()
