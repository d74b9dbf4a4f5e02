"""Multi-GPU drivers for the Fourier LLF hot path.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing, NCCL
over NVLink for the single exchange step the path has.

* Frame data-parallel (config 5): frames are independent problems; each rank
  filters a contiguous slice of the batch with one batched plan.  No
  collective on the data path.
* Order sharding (config 3): the work units are (channel, order k) pairs.
  Rank r gets a contiguous, balanced run of units (channel-major), builds only
  its orders' Gaussian Fourier pyramids (plus G, replicated) and collapses its
  partial output locally -- the collapse of Eq. 4 is linear, so
  the full output is I + sum over ranks of the partials.  The rank owning
  order 1 of a channel adds I (``include_base``).  One NCCL reduce (sum, fp32)
  per channel to rank 0, issued as soon as that channel's partial is ready so
  it overlaps the next channel's compute.

The partitioning and the reduce schedule are plain host logic (tested on CPU
with the gloo backend, world size 2); the per-unit compute is whatever
``partial_fn`` the caller passes -- on GPU, a libfllf plan per segment
(:func:`gpu_partial_fn`).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List


class _nvtx:
    """NVTX range (torch.cuda.nvtx) when CUDA is present; a no-op on CPU-only hosts."""

    def __init__(self, msg: str):
        self.msg = msg
        self.on = False

    def __enter__(self):
        try:
            import torch
            if torch.cuda.is_available():
                torch.cuda.nvtx.range_push(self.msg)
                self.on = True
        except Exception:  # pragma: no cover
            pass
        return self

    def __exit__(self, *exc):
        if self.on:
            import torch
            torch.cuda.nvtx.range_pop()


def frame_partition(n_frames: int, world: int, rank: int) -> tuple[int, int]:
    """(first frame, count) of rank's contiguous, balanced slice."""
    base, extra = divmod(n_frames, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


@dataclass(frozen=True)
class Segment:
    channel: int
    k_begin: int      # 1-based, inclusive
    k_end: int        # exclusive
    include_base: bool
    nch: int = 1      # channels channel .. channel+nch-1 with this order range (batch_channels)


def order_partition(channels: int, K: int, world: int) -> List[List[Segment]]:
    """Split the channels*K (channel, order) units into `world` contiguous runs
    whose sizes differ by at most one; express each run as per-channel order
    ranges.  include_base marks the segment that owns order 1 of a channel."""
    total = channels * K
    out: List[List[Segment]] = []
    for r in range(world):
        first, count = frame_partition(total, world, r)
        segs: List[Segment] = []
        u = first
        while u < first + count:
            c, k0 = divmod(u, K)
            take = min(K - k0, first + count - u)
            segs.append(Segment(c, k0 + 1, k0 + 1 + take, k0 == 0))
            u += take
        out.append(segs)
    return out


def channel_runs(segs: List[Segment]) -> List[Segment]:
    """Merge consecutive channels that carry the same order range into one
    segment with nch > 1 (one batched plan instead of one plan per channel)."""
    runs: List[Segment] = []
    for s in sorted(segs, key=lambda x: x.channel):
        r = runs[-1] if runs else None
        if (r is not None and r.channel + r.nch == s.channel and (r.k_begin, r.k_end, r.include_base) ==
                (s.k_begin, s.k_end, s.include_base)):
            runs[-1] = Segment(r.channel, r.k_begin, r.k_end, r.include_base, r.nch + s.nch)
        else:
            runs.append(s)
    return runs


def sharded_filter(partial_fn: Callable, out, channels: int, K: int, group=None, dst: int = 0,
                   overlap: bool = True, batch_channels: bool = False):
    """Order-sharded Fourier LLF with one reduce per channel.

    partial_fn(segment, out_channel) must write this rank's partial output of
    `segment` INTO out_channel (a (H, W) view of `out`); channels this rank
    has no unit of are zero-filled here.  `out` is (channels, H, W) on the
    rank's device; after the call, rank `dst` holds the full output.
    batch_channels: consecutive channels with the same order range go to
    partial_fn as ONE segment (nch > 1) with the (nch, H, W) view -- e.g. all
    three channels on a single rank as one batched plan; each channel's
    reduce is issued once its run is computed.
    Returns the list of async work handles already waited on.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = order_partition(channels, K, world)[rank]
    if batch_channels:
        runs = channel_runs(mine)
        owned = {c for r in runs for c in range(r.channel, r.channel + r.nch)}
        works = []
        nxt = 0  # next channel to reduce: every rank issues the reduces in channel order

        def reduce_upto(last):
            nonlocal nxt
            while nxt <= last:
                if nxt not in owned:
                    out[nxt].zero_()
                with _nvtx(f"fllf reduce channel {nxt}"):
                    w = dist.reduce(out[nxt], dst=dst, op=dist.ReduceOp.SUM, group=group, async_op=overlap)
                if overlap:
                    works.append(w)
                nxt += 1

        for r in runs:
            # the run's kernels are enqueued; its channels' reduces go out now, so
            # they wait only for the work queued so far and overlap the next run
            with _nvtx(f"fllf partial channels {r.channel}..{r.channel + r.nch - 1}"):
                partial_fn(r, out[r.channel:r.channel + r.nch])
            reduce_upto(r.channel + r.nch - 1)
        reduce_upto(channels - 1)
        for w in works:
            w.wait()
        return works
    by_ch = {}
    for s in mine:
        by_ch.setdefault(s.channel, []).append(s)
    works = []
    for c in range(channels):
        segs = by_ch.get(c, [])
        if not segs:
            out[c].zero_()
        for i, s in enumerate(segs):
            if i == 0:
                partial_fn(s, out[c])
            else:  # two ranges of one channel on one rank cannot happen with contiguous runs
                raise AssertionError("non-contiguous order range within a channel")
        w = dist.reduce(out[c], dst=dst, op=dist.ReduceOp.SUM, group=group, async_op=overlap)
        if overlap:
            works.append(w)
    for w in works:
        w.wait()
    return works


def gpu_partial_fn(img, levels: int, K: int, T: float, sigma_r: float, m: float):
    """partial_fn backed by libfllf: one plan per segment (created once, cached),
    reading channel `segment.channel` of the (C, H, W) CUDA tensor `img`."""
    from . import fllf as F

    H, W = img.shape[-2:]
    plans = {}

    def fn(seg: Segment, out_c):
        key = (seg.channel, seg.k_begin, seg.k_end, seg.include_base, seg.nch)
        p = plans.get(key)
        if p is None:
            p = F.Plan(H, W, levels, K, T, sigma_r, m, k_begin=seg.k_begin, k_end=seg.k_end,
                       include_base=seg.include_base, batch=seg.nch)
            plans[key] = p
        src = img[seg.channel] if seg.nch == 1 and out_c.dim() == 2 else img[seg.channel:seg.channel + seg.nch]
        p.filter(src, out_c)

    fn.plans = plans
    return fn


class P2PCombine:
    """Order sharding with the combine fused into the level-0 apply (a7): the
    owner rank allocates the (channels, H, W) output with fllf_ipc_alloc and
    shares its CUDA IPC handle; every rank maps it and its partial plans add
    their outputs straight into it with fllf_apply_accumulate (hardware atomics;
    over NVLink when the owner is another GPU) -- no partial buffers, no
    separate reduce.  Per call: owner zeroes, barrier, partials, barrier.

    img: (channels, H, W) CUDA tensor on this rank's device (every rank holds
    the input).  run() returns the output tensor on the owner, None elsewhere.
    The host logic (partition, handle exchange, ordering) is plain
    torch.distributed and runs under gloo as well."""

    def __init__(self, img, levels: int, K: int, T: float, sigma_r: float, m: float, group=None, dst: int = 0):
        import torch
        import torch.distributed as dist

        from . import fllf as F
        self.F, self.dist, self.torch = F, dist, torch
        self.group, self.dst = group, dst
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.img = img
        C, H, W = img.shape
        self.shape = (C, H, W)
        self.device = img.device.index
        nbytes = C * H * W * 4
        if self.rank == dst:
            self.ptr, handle = F.ipc_alloc(nbytes)
            self.owned = True
        else:
            self.ptr, handle, self.owned = None, None, False
        obj = [handle]
        dist.broadcast_object_list(obj, src=dst, group=group)
        if not self.owned:
            self.ptr = F.ipc_open(obj[0])
        self.out = F.device_view(self.ptr, (C, H, W), (H * W, W, 1), self.device)
        runs = channel_runs(order_partition(C, K, self.world)[self.rank])
        self.jobs = []
        for r in runs:
            p = F.Plan(H, W, levels, K, T, sigma_r, m, k_begin=r.k_begin, k_end=r.k_end,
                       include_base=r.include_base, batch=r.nch)
            self.jobs.append((r, p))

    def run(self):
        torch, dist, F = self.torch, self.dist, self.F
        if self.owned:
            self.out.zero_()
            torch.cuda.synchronize()
        dist.barrier(group=self.group)
        for r, p in self.jobs:
            src = self.img[r.channel:r.channel + r.nch]
            p.build(src)
            F.fllf_apply_accumulate(p.handle, self.out[r.channel:r.channel + r.nch])
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        return self.out if self.owned else None

    def close(self):
        for _, p in self.jobs:
            p.close()
        self.jobs = []
        if self.ptr is not None:
            self.torch.cuda.synchronize()
            (self.F.ipc_free if self.owned else self.F.ipc_close)(self.ptr)
            self.ptr = None


# ------------------------------------------------------------------ NEXT-1
# Row-band split with per-level halo exchange (north star: "Large frames can
# instead be split into row bands with halo exchange").  Every level of both
# passes only couples neighbouring rows: the build of level l+1 reads fine rows
# 2o-2 .. 2o+2 (Eq. 1, 5-tap), the apply of level l reads the coarse rows
# r-1 .. r+1 of Z_{l+1} and D_{l+1} (up-sampling).  A band therefore needs two
# halo rows per side of G_l, Z_l (after the build of level l) and of D_l
# (after the apply of level l), exchanged between neighbouring bands only --
# no collective over the whole frame, and the traffic per level is
# 4 rows x (2K+2) planes x W_l x 4 B, independent of the number of bands.

BAND_G, BAND_Z, BAND_D = 0, 1, 2


def band_partition(H: int, levels: int, world: int) -> List[tuple]:
    """Contiguous row bands [row_begin, row_end) with boundaries at multiples of
    2^(levels-1) (so every level's band is a whole number of rows) and at least
    2 own rows per band at the coarsest level; balanced to one alignment unit."""
    align = 1 << (levels - 1)
    units = -(-H // align)
    if units < 2 * world:
        raise ValueError(f"{H} rows at {levels} levels allow at most {units // 2} bands")
    out = []
    for r in range(world):
        f, c = frame_partition(units, world, r)
        out.append((f * align, min((f + c) * align, H)))
    return out


def band_level_rows(H: int, levels: int, band: tuple, level: int) -> tuple:
    """The band's own rows [b, e) at `level` (global indices, ceil-halving)."""
    h = H
    for _ in range(level):
        h = (h + 1) // 2
    rb, re_ = band
    return rb >> level, (h if re_ == H else re_ >> level)


def band_schedule(levels: int) -> list:
    """Per-level steps of one band: ('build', l) makes level l+1; ('xchg', l,
    kinds) refreshes the halo rows of level l; ('apply', l) is the apply of l."""
    steps = []
    for l in range(levels - 1):
        steps.append(("build", l))
        steps.append(("xchg", l + 1, (BAND_G, BAND_Z)))
    for l in range(levels - 2, -1, -1):
        if l + 1 < levels - 1:
            steps.append(("xchg", l + 1, (BAND_D,)))
        steps.append(("apply", l))
    return steps


def halo_slices(first_row: int, rows: int, own: tuple):
    """Row indices (into a stored-rows view starting at global `first_row`) of
    the top halo, the bottom halo, the first two own rows and the last two."""
    b, e = own
    top = slice(0, b - first_row)
    bot = slice(e - first_row, rows)
    n_top, n_bot = top.stop - top.start, bot.stop - bot.start
    send_up = slice(b - first_row, b - first_row + 2)
    send_dn = slice(e - first_row - 2, e - first_row)
    return top, bot, send_up, send_dn, n_top, n_bot


def exchange_halos(view, first_row: int, own: tuple, group=None, up: int = None, down: int = None):
    """Fill the halo rows of `view` (planes, rows, floats: a band's stored rows of
    one plane kind and level) from the neighbouring ranks `up` / `down` (None at
    the frame border), sending them this band's edge rows; NCCL / gloo p2p."""
    import torch.distributed as dist

    top, bot, send_up, send_dn, n_top, n_bot = halo_slices(first_row, view.shape[1], own)
    ops, recv = [], []
    if up is not None:
        ops.append(dist.P2POp(dist.isend, view[:, send_up].contiguous(), up, group))
        buf = view.new_empty((view.shape[0], n_top, view.shape[2]))
        ops.append(dist.P2POp(dist.irecv, buf, up, group))
        recv.append((top, buf))
    if down is not None:
        ops.append(dist.P2POp(dist.isend, view[:, send_dn].contiguous(), down, group))
        buf = view.new_empty((view.shape[0], n_bot, view.shape[2]))
        ops.append(dist.P2POp(dist.irecv, buf, down, group))
        recv.append((bot, buf))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for sl, buf in recv:
        view[:, sl] = buf


class GpuBand:
    """One rank's band: a libfllf plan over rows [row_begin, row_end) of an
    H x W frame and the per-level execution of `band_schedule`."""

    def __init__(self, H, W, levels, K, T, sigma_r, m, band, device=0):
        from . import fllf as F
        self.F, self.H, self.levels, self.band, self.device = F, H, levels, band, device
        self.plan = F.Plan(H, W, levels, K, T, sigma_r, m, row_begin=band[0], row_end=band[1])

    def view(self, level, kind):
        return self.F.band_rows_view(self.plan.handle, level, kind, self.device)

    def own(self, level):
        return band_level_rows(self.H, self.levels, self.band, level)

    def run_step(self, step, img_ptr, img_pitch, out_ptr, out_pitch, stream=None):
        if step[0] == "build":
            self.F.fllf_build_level(self.plan.handle, img_ptr, img_pitch, step[1], stream)
        elif step[0] == "apply":
            self.F.fllf_apply_level(self.plan.handle, out_ptr, out_pitch, step[1], stream=stream)

    def close(self):
        self.plan.close()


def band_filter(gb: GpuBand, img_band, out_band, group=None):
    """Row-band Fourier LLF on this rank.  img_band: CUDA (rows, W) tensor holding
    the band's rows plus the 2 rows above / below it (where they exist);
    out_band: (row_end - row_begin, W).  Neighbours are ranks rank-1 / rank+1."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    up = rank - 1 if rank > 0 else None
    down = rank + 1 if rank + 1 < world else None
    top_in = gb.band[0] - max(0, gb.band[0] - 2)
    ipitch = img_band.stride(0) * 4
    iptr = img_band.data_ptr() + top_in * ipitch
    for step in band_schedule(gb.levels):
        if step[0] == "xchg":
            with _nvtx(f"fllf halo exchange level {step[1]}"):
                for kind in step[2]:
                    v, first = gb.view(step[1], kind)
                    exchange_halos(v, first, gb.own(step[1]), group, up, down)
        else:
            gb.run_step(step, iptr, ipitch, out_band.data_ptr(), out_band.stride(0) * 4)


def band_filter_local(bands: list, img, out):
    """All bands of one frame on the current GPU (single-process emulation of
    band_filter, for tests and for one GPU): the same per-level schedule, the
    halo exchange done as device copies between the bands' stored rows.
    img / out: CUDA (H, W) tensors of the whole frame."""
    H = img.shape[0]
    levels = bands[0].levels
    ipitch, opitch = img.stride(0) * 4, out.stride(0) * 4
    for step in band_schedule(levels):
        if step[0] == "xchg":
            l = step[1]
            for kind in step[2]:
                views = [gb.view(l, kind) for gb in bands]
                for i in range(len(bands) - 1):
                    (vu, fu), (vd, fd) = views[i], views[i + 1]
                    ou, od = bands[i].own(l), bands[i + 1].own(l)
                    _, bot_u, _, send_dn_u, _, _ = halo_slices(fu, vu.shape[1], ou)
                    top_d, _, send_up_d, _, _, _ = halo_slices(fd, vd.shape[1], od)
                    vu[:, bot_u] = vd[:, send_up_d]
                    vd[:, top_d] = vu[:, send_dn_u]
        else:
            for gb in bands:
                rb = gb.band[0]
                gb.run_step(step, img.data_ptr() + rb * ipitch, ipitch, out.data_ptr() + rb * opitch, opitch)
