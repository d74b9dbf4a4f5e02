"""Multi-process host logic of the multi-GPU drivers, on CPU with gloo
(world size 2, 127.0.0.1).  The per-unit compute is the fp64 oracle here (test
infrastructure); on GPU it is a libfllf plan (paper_2206_04681_b200.dist.gpu_partial_fn)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_04681_b200.dist import Segment, frame_partition, order_partition, sharded_filter


def test_frame_partition_covers_all():
    for n in (1, 7, 64):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                f, c = frame_partition(n, world, r)
                seen += list(range(f, f + c))
                assert abs(c - n / world) < 1
            assert seen == list(range(n))


@pytest.mark.parametrize("C,K", [(3, 10), (1, 8), (3, 1), (2, 16)])
@pytest.mark.parametrize("world", [1, 2, 4, 8, 13])
def test_order_partition_properties(C, K, world):
    parts = order_partition(C, K, world)
    units = [(s.channel, k) for segs in parts for s in segs for k in range(s.k_begin, s.k_end)]
    assert sorted(units) == [(c, k) for c in range(C) for k in range(1, K + 1)]
    sizes = [sum(s.k_end - s.k_begin for s in segs) for segs in parts]
    assert max(sizes) - min(sizes) <= 1
    for c in range(C):
        assert sum(1 for segs in parts for s in segs if s.channel == c and s.include_base) == 1
    for segs in parts:                       # at most one range per channel per rank
        chans = [s.channel for s in segs]
        assert len(chans) == len(set(chans))


def test_config3_balance_at_8():
    parts = order_partition(3, 10, 8)       # 30 units -> 4,4,4,4,4,4,3,3
    assert sorted(sum(s.k_end - s.k_begin for s in p) for p in parts) == [3, 3, 4, 4, 4, 4, 4, 4]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, img, args, result_path):
    from oracle import fllf_oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    levels, K, T, sig, m = args
    C, H, W = img.shape
    out = torch.zeros((C, H, W), dtype=torch.float64)

    batch = world == 1 or os.environ.get("FLLF_TEST_BATCH_CH") == "1"

    def partial_fn(seg: Segment, out_c):
        views = out_c if batch else out_c[None]
        assert views.shape[0] == seg.nch and (batch or seg.nch == 1)
        for i in range(seg.nch):
            c = seg.channel + i
            part = O.fourier_llf(img[c], levels, K, T, sig, m, k_range=(seg.k_begin, seg.k_end),
                                 include_base=False)
            if seg.include_base:
                part = part + img[c]
            views[i].copy_(torch.from_numpy(part))

    sharded_filter(partial_fn, out, C, K, batch_channels=batch)
    if rank == 0:
        np.save(result_path, out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,batch", [(1, True), (2, False), (2, True), (3, True)])
def test_sharded_filter_gloo_equals_full(tmp_path, monkeypatch, world, batch):
    """Order sharding with one reduce per channel.  batch: consecutive channels
    with one order range run as one batched call, and each run's reduces are
    issued right after it (every rank in channel order, zero-filled channels
    without units included) -- world 3 gives ranks owning different channel
    sets, so a rank-dependent reduce order would hang or mix channels."""
    monkeypatch.setenv("FLLF_TEST_BATCH_CH", "1" if batch else "0")
    rng = np.random.default_rng(3)
    img = rng.uniform(0, 255, (3, 24, 21))
    args = (3, 5, 510.0, 20.0, 2.0)
    res = str(tmp_path / "out.npy")
    mp.spawn(_worker, args=(world, _free_port(), img, args, res), nprocs=world, join=True)
    from oracle import fllf_oracle as O
    full = np.stack([O.fourier_llf(img[c], *args) for c in range(3)])
    assert np.abs(np.load(res) - full).max() <= 1e-9


def test_channel_runs():
    from paper_2206_04681_b200.dist import channel_runs
    for C, K, world in [(3, 10, 1), (3, 10, 2), (3, 10, 3), (3, 10, 8), (4, 6, 3), (5, 4, 2)]:
        parts = order_partition(C, K, world)
        for segs in parts:
            runs = channel_runs(segs)
            # same units, channels covered once, merged runs share one order range
            cov = [c for r in runs for c in range(r.channel, r.channel + r.nch)]
            assert sorted(cov) == sorted(s.channel for s in segs)
            for r in runs:
                assert any(s.channel == r.channel and (s.k_begin, s.k_end) == (r.k_begin, r.k_end) for s in segs)
    assert [r.nch for r in channel_runs(order_partition(3, 10, 1)[0])] == [3]


# ---------------------------------------------------------------- NEXT-1
def test_band_partition_properties():
    from paper_2206_04681_b200.dist import band_level_rows, band_partition
    for H, levels, world in [(2160, 7, 8), (1080, 6, 4), (517, 3, 7), (300, 5, 3), (128, 2, 2)]:
        bands = band_partition(H, levels, world)
        align = 1 << (levels - 1)
        assert bands[0][0] == 0 and bands[-1][1] == H
        for (a, b), (c, d) in zip(bands, bands[1:]):
            assert b == c and b % align == 0
        h = H
        for l in range(levels):
            rows = [band_level_rows(H, levels, bd, l) for bd in bands]
            assert rows[0][0] == 0 and rows[-1][1] == h
            assert all(e - b >= 2 for b, e in rows)
            assert all(r1[1] == r2[0] for r1, r2 in zip(rows, rows[1:]))
            h = (h + 1) // 2
    with pytest.raises(ValueError):
        band_partition(100, 6, 4)


def _band_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2206_04681_b200.dist import band_level_rows, band_partition, exchange_halos
    H, levels, W = 300, 4, 5
    band = band_partition(H, levels, world)[rank]
    ok = True
    for l in range(1, levels):
        b, e = band_level_rows(H, levels, band, l)
        hl = H
        for _ in range(l):
            hl = (hl + 1) // 2
        lo, hi = max(0, b - 2), min(hl, e + 2)
        # stored rows: own rows hold their global row index, halos -1
        v = torch.full((2, hi - lo, W), -1.0)
        for r in range(b, e):
            v[:, r - lo] = float(r)
        exchange_halos(v, lo, (b, e), None, rank - 1 if rank > 0 else None, rank + 1 if rank + 1 < world else None)
        expect = torch.arange(lo, hi, dtype=torch.float32)[None, :, None].expand_as(v)
        ok = ok and bool(torch.equal(v, expect))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_band_halo_exchange_gloo(world):
    """Every halo row a band stores equals the neighbour's row of the same global index."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ps = [ctx.Process(target=_band_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert all(res.values()), res
