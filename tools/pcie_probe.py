"""Host<->device copy bandwidth on this box (pinned memory): H2D alone, D2H
alone, both at once on two streams, H2D split over several streams, and the
same after pinning the process to the GPU's NUMA-local CPUs -- the ceiling of
the streaming end-to-end path (fllf_filter_host_frames).
    python tools/pcie_probe.py [--local]
"""
import os
import sys

import torch

FR = 8294400  # one 1080x1920 fp32 frame


def gpu_local_cpus(dev=0):
    bus = torch.cuda.get_device_properties(dev).pci_bus_id if hasattr(torch.cuda.get_device_properties(dev), "pci_bus_id") else None
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        bus = pynvml.nvmlDeviceGetPciInfo(h).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
    except Exception:
        pass
    if not bus:
        return None, None
    bus = bus.lower()
    if bus.count(":") == 2 and len(bus.split(":")[0]) == 8:
        bus = bus[4:]
    base = f"/sys/bus/pci/devices/{bus}"
    try:
        cl = open(base + "/local_cpulist").read().strip()
        node = open(base + "/numa_node").read().strip()
    except OSError:
        return bus, None
    cpus = set()
    for part in cl.split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return (bus, node), cpus


def main():
    torch.cuda.init()
    info, cpus = gpu_local_cpus()
    print("gpu pci / numa node:", info, "local cpus:", (min(cpus), max(cpus), len(cpus)) if cpus else None,
          "affinity now:", len(os.sched_getaffinity(0)), flush=True)
    if "--local" in sys.argv and cpus:
        os.sched_setaffinity(0, cpus & os.sched_getaffinity(0) or cpus)
        print("pinned to", len(os.sched_getaffinity(0)), "local cpus", flush=True)
    n = 20
    h_in = torch.empty(FR // 4, dtype=torch.float32).pin_memory()
    h_in.fill_(1.0)
    h_out = torch.empty(FR // 4, dtype=torch.float32).pin_memory()
    h_out.fill_(1.0)
    d_a = torch.empty(FR // 4, dtype=torch.float32, device="cuda")
    d_b = torch.empty(FR // 4, dtype=torch.float32, device="cuda")
    ss = [torch.cuda.Stream() for _ in range(5)]

    def run(h2d_split, d2h):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for s in ss:
            s.wait_event(a)
        for _ in range(n):
            if h2d_split:
                c = FR // 4 // h2d_split
                for j in range(h2d_split):
                    with torch.cuda.stream(ss[j]):
                        d_a[j * c:(j + 1) * c].copy_(h_in[j * c:(j + 1) * c], non_blocking=True)
            if d2h:
                with torch.cuda.stream(ss[4]):
                    h_out.copy_(d_b, non_blocking=True)
        for s in ss:
            e = torch.cuda.Event()
            e.record(s)
            torch.cuda.current_stream().wait_event(e)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        return ms / n * 1e3, FR / (ms / n / 1e3) / 1e9

    for name, h, d in (("H2D", 1, 0), ("H2D x2 streams", 2, 0), ("H2D x4 streams", 4, 0), ("D2H", 0, 1),
                       ("both", 1, 1), ("both, H2D x4", 4, 1)):
        run(h, d)
        us, gbs = run(h, d)
        print(f"{name}: {us:.1f} us per 8.29 MB frame, {gbs:.1f} GB/s per direction", flush=True)


if __name__ == "__main__":
    main()
