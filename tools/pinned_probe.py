"""Pinned-host-memory flavours vs copy bandwidth (one 1080p fp32 frame):
torch .pin_memory(), torch.empty(pin_memory=True), and cudaHostAlloc through
libfllf's fllf_host_alloc -- H2D, D2H and both at once on two streams."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

FR = 8294400
n = 20


def bench(h_in, h_out):
    d_a = torch.empty(FR // 4, device="cuda")
    d_b = torch.empty(FR // 4, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, h, d in (("H2D", 1, 0), ("D2H", 0, 1), ("both", 1, 1)):
        for rep in range(2):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s1.wait_event(a)
            s2.wait_event(a)
            for _ in range(n):
                if h:
                    with torch.cuda.stream(s1):
                        d_a.copy_(h_in, non_blocking=True)
                if d:
                    with torch.cuda.stream(s2):
                        h_out.copy_(d_b, non_blocking=True)
            for s in (s1, s2):
                e = torch.cuda.Event()
                e.record(s)
                torch.cuda.current_stream().wait_event(e)
            b.record()
            torch.cuda.synchronize()
        res[name] = a.elapsed_time(b) / n * 1e3
    return res


def main():
    torch.cuda.init()
    x = torch.empty(FR // 4).pin_memory(); x.fill_(1)
    y = torch.empty(FR // 4).pin_memory(); y.fill_(1)
    print("torch .pin_memory()        ", {k: f"{v:.0f} us" for k, v in bench(x, y).items()}, flush=True)
    x = torch.empty(FR // 4, pin_memory=True); x.fill_(1)
    y = torch.empty(FR // 4, pin_memory=True); y.fill_(1)
    print("torch.empty(pin_memory=True)", {k: f"{v:.0f} us" for k, v in bench(x, y).items()}, flush=True)
    from paper_2206_04681_b200 import fllf as F
    if hasattr(F, "host_empty"):
        x = F.host_empty((FR // 4,)); x.fill_(1)
        y = F.host_empty((FR // 4,)); y.fill_(1)
        print("fllf_host_alloc (cudaHostAlloc)", {k: f"{v:.0f} us" for k, v in bench(x, y).items()}, flush=True)
    cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    if cudart is not None:
        p1, p2 = ctypes.c_void_p(), ctypes.c_void_p()
        cudart.cudaHostAlloc(ctypes.byref(p1), ctypes.c_size_t(FR), 0)
        cudart.cudaHostAlloc(ctypes.byref(p2), ctypes.c_size_t(FR), 0)
        buf1 = (ctypes.c_float * (FR // 4)).from_address(p1.value)
        buf2 = (ctypes.c_float * (FR // 4)).from_address(p2.value)
        x = torch.frombuffer(buf1, dtype=torch.float32); x.fill_(1)
        y = torch.frombuffer(buf2, dtype=torch.float32); y.fill_(1)
        print("cudart cudaHostAlloc (ctypes)", {k: f"{v:.0f} us" for k, v in bench(x, y).items()}, flush=True)


if __name__ == "__main__":
    main()


def raw_cudart():
    """The same copies through cudart directly (no torch copy_)."""
    import time
    cudart = ctypes.CDLL("libcudart.so.12")
    h, d = ctypes.c_void_p(), ctypes.c_void_p()
    cudart.cudaHostAlloc(ctypes.byref(h), ctypes.c_size_t(FR), 0)
    cudart.cudaMalloc(ctypes.byref(d), ctypes.c_size_t(FR))
    ctypes.memset(h, 1, FR)
    for kind, name in ((1, "H2D"), (2, "D2H")):
        src, dst = (h, d) if kind == 1 else (d, h)
        cudart.cudaMemcpy(dst, src, ctypes.c_size_t(FR), kind)
        t = time.perf_counter()
        for _ in range(n):
            cudart.cudaMemcpyAsync(dst, src, ctypes.c_size_t(FR), kind, None)
        cudart.cudaDeviceSynchronize()
        dt = (time.perf_counter() - t) / n
        print(f"raw cudart {name}: {dt * 1e6:.0f} us per frame ({FR / dt / 1e9:.1f} GB/s)", flush=True)


if __name__ == "__main__" and "--raw" in sys.argv:
    raw_cudart()
