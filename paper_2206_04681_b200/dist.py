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


def sharded_filter(partial_fn: Callable, out, channels: int, K: int, group=None, dst: int = 0,
                   overlap: bool = True):
    """Order-sharded Fourier LLF with one reduce per channel.

    partial_fn(segment, out_channel) must write this rank's partial output of
    `segment` INTO out_channel (a (H, W) view of `out`); channels this rank
    has no unit of are zero-filled here.  `out` is (channels, H, W) on the
    rank's device; after the call, rank `dst` holds the full output.
    Returns the list of async work handles already waited on.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = order_partition(channels, K, world)[rank]
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
        key = (seg.channel, seg.k_begin, seg.k_end, seg.include_base)
        p = plans.get(key)
        if p is None:
            p = F.Plan(H, W, levels, K, T, sigma_r, m, k_begin=seg.k_begin, k_end=seg.k_end,
                       include_base=seg.include_base)
            plans[key] = p
        p.filter(img[seg.channel], out_c)

    fn.plans = plans
    return fn
