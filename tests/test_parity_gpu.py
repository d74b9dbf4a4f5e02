"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle.

Bar (BASELINE.json north star): max |GPU - oracle| <= 2e-3 on the 0-255 scale,
fp32 device vs fp64 oracle, on the same seeded inputs.  Pyramid planes are
checked per stage with tolerances derived from fp32 rounding (DESIGN.md
"Tolerances").  Everything here calls libfllf via the ctypes binding.
"""
import numpy as np
import pytest
import torch

from oracle import fllf_oracle as O
from paper_2206_04681_b200 import synth

pytestmark = pytest.mark.gpu

TOL_OUT = 2e-3      # north star, output on the 0-255 scale
TOL_G = 2e-4        # G_l planes (values <= 255, fp32 sums of 5x5 taps)
TOL_Z = 2e-5        # Z_{l,k} planes (|values| <= 1; sincos + recurrence error)


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_04681_b200 import fllf
    return fllf


def gpu_run(F, img, levels, K, T, sigma_r=30.0, m=1.0, mode=0, a_k=None, smap=None, mmap=None,
            k_begin=0, k_end=0, include_base=True, pitch_pad=0):
    """img: (H, W) or (B, H, W) float32 numpy.  Returns float64 numpy output."""
    x = np.asarray(img, dtype=np.float32)
    B = x.shape[0] if x.ndim == 3 else 1
    H, W = x.shape[-2:]
    if pitch_pad:
        buf = torch.zeros((B, H, W + pitch_pad), dtype=torch.float32, device="cuda")
        buf[:, :, :W] = torch.from_numpy(x.reshape(B, H, W)).cuda()
        d_in = buf[:, :, :W]
    else:
        d_in = torch.from_numpy(x.reshape(B, H, W)).cuda()
    d_out = torch.full((B, H, W), float("nan"), dtype=torch.float32, device="cuda")
    with F.Plan(H, W, levels, K, T, sigma_r, m, batch=B, k_begin=k_begin, k_end=k_end,
                include_base=include_base) as p:
        p.build(d_in)
        kw = {}
        if mode == F.FLLF_COEFFS:
            kw = dict(mode=mode, a_k=a_k)
        elif mode == F.FLLF_MAPS:
            kw = dict(mode=mode, sigma_map=torch.from_numpy(np.asarray(smap, np.float32)).cuda(),
                      m_map=torch.from_numpy(np.asarray(mmap, np.float32)).cuda())
        p.apply(d_out, **kw)
        torch.cuda.synchronize()
        assert p.launches >= 1
    out = d_out.cpu().numpy().astype(np.float64)
    return out if x.ndim == 3 else out[0]


def maxerr(a, b):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max())


# --------------------------------------------------------------- per stage
@pytest.mark.parametrize("shape,levels,K,T", [((256, 256), 4, 4, 510.0), ((37, 23), 3, 5, 510.0),
                                              ((135, 17), 4, 9, 405.9), ((70, 97), 5, 12, 510.0)])
def test_pyramid_planes(F, shape, levels, K, T):
    img = synth.uniform_image(*shape, seed=101)
    G, Ct, St = O.fourier_llf_pyramids(img.astype(np.float64), levels, K, T)
    d_in = torch.from_numpy(img).cuda()
    with F.Plan(shape[0], shape[1], levels, K, T) as p:
        p.build(d_in)
        for l in range(1, levels):
            h, w = p.level_dims(l)
            assert (h, w) == G[l].shape
            g = torch.empty((h, w), dtype=torch.float32, device="cuda")
            p.read_pyramid(0, l, 0, g)
            assert maxerr(g.cpu().numpy(), G[l]) <= TOL_G, (l, "G")
            for k in range(1, K + 1):
                z = torch.empty((h, 2 * w), dtype=torch.float32, device="cuda")
                p.read_pyramid(0, l, k, z)
                z = z.cpu().numpy().astype(np.float64)
                assert maxerr(z[:, 0::2], St[k - 1][l]) <= TOL_Z, (l, k, "S")
                assert maxerr(z[:, 1::2], Ct[k - 1][l]) <= TOL_Z, (l, k, "C")


# ------------------------------------------------------------- end to end
def test_config1_full(F):
    c = synth.CONFIGS[1]
    img = synth.config1_image()
    ref = O.fourier_llf(img.astype(np.float64), c["levels"], c["K"], c["T"], c["sigma_r"], c["m"])
    out = gpu_run(F, img, c["levels"], c["K"], c["T"], c["sigma_r"], c["m"])
    assert maxerr(out, ref) <= TOL_OUT


@pytest.mark.parametrize("shape,levels,K,T,sig,m,pad", [
    ((37, 23), 3, 5, 510.0, 30.0, -1.5, 0),      # odd sizes, smoothing gain, unaligned pitch
    ((50, 71), 4, 8, 510.0, 20.0, 3.0, 0),
    ((9, 13), 3, 3, 405.9, 30.0, 7.0, 0),        # tiny: coarsest level 3x4
    ((121, 300), 6, 16, 510.0, 10.0, 4.0, 5),    # ragged + padded pitch, K=16
    ((64, 33), 2, 10, 405.9, 30.0, 7.0, 0),      # 2 levels (paper's "2-layer")
    ((259, 130), 7, 1, 510.0, 60.0, 2.0, 3),     # K=1
])
def test_ragged_end_to_end(F, shape, levels, K, T, sig, m, pad):
    img = synth.uniform_image(*shape, seed=7 + K)
    ref = O.fourier_llf(img.astype(np.float64), levels, K, T, sig, m)
    out = gpu_run(F, img, levels, K, T, sig, m, pitch_pad=pad)
    assert maxerr(out, ref) <= TOL_OUT


def test_constant_and_zero_gain(F):
    C = np.full((45, 62), 93.5, np.float32)
    assert maxerr(gpu_run(F, C, 4, 8, 510.0, 30.0, 3.0), C) <= 1e-4
    img = synth.uniform_image(45, 62, seed=3)
    assert maxerr(gpu_run(F, img, 4, 8, 510.0, 30.0, 0.0), img) <= 1e-4


def test_coeffs_mode_and_reapply(F):
    """Build once, apply with two coefficient sets."""
    img = synth.config1_image(seed=1001, H=96, W=80)
    K, T = 6, 510.0
    a1 = O.fourier_coefficients(K, T, 30.0, 2.0)["a"]
    a2 = np.linspace(3.0, -1.0, K)                       # any odd detail term
    r1 = O.fourier_llf(img.astype(np.float64), 4, K, T, a=a1)
    r2 = O.fourier_llf(img.astype(np.float64), 4, K, T, a=a2)
    d_in = torch.from_numpy(img).cuda()
    o = torch.empty_like(d_in)
    with F.Plan(96, 80, 4, K, T, 30.0, 2.0) as p:
        p.build(d_in)
        p.apply(o, mode=F.FLLF_COEFFS, a_k=a1)
        assert maxerr(o.cpu().numpy(), r1) <= TOL_OUT
        p.apply(o, mode=F.FLLF_COEFFS, a_k=a2)
        assert maxerr(o.cpu().numpy(), r2) <= TOL_OUT
        p.apply(o)                                       # SCALAR == a1
        assert maxerr(o.cpu().numpy(), r1) <= TOL_OUT


def test_maps_mode(F):
    H, W = 90, 131
    img = synth.uniform_image(H, W, seed=21)
    rng = np.random.default_rng(5)
    s = rng.uniform(10.0, 60.0, (H, W)).astype(np.float32)
    mm = rng.uniform(0.5, 4.0, (H, W)).astype(np.float32)
    ref = O.fourier_llf(img.astype(np.float64), 5, 12, 510.0, sigma_map=s.astype(np.float64),
                        m_map=mm.astype(np.float64))
    out = gpu_run(F, img, 5, 12, 510.0, mode=F.FLLF_MAPS, smap=s, mmap=mm)
    assert maxerr(out, ref) <= TOL_OUT
    # constant maps == scalar mode
    cs, cm = np.full((H, W), 25.0, np.float32), np.full((H, W), 2.5, np.float32)
    o1 = gpu_run(F, img, 5, 12, 510.0, mode=F.FLLF_MAPS, smap=cs, mmap=cm)
    o2 = gpu_run(F, img, 5, 12, 510.0, 25.0, 2.5)
    assert maxerr(o1, o2) <= 1e-3


def test_order_partition(F):
    """Order sharding (config 3 layout): partials over a partition of 1..K plus I == full."""
    img = synth.uniform_image(77, 90, seed=31)
    K, lev = 10, 4
    full = O.fourier_llf(img.astype(np.float64), lev, K, 510.0, 20.0, 2.0)
    parts = []
    for kb, ke in [(1, 4), (4, 8), (8, 11)]:
        part = gpu_run(F, img, lev, K, 510.0, 20.0, 2.0, k_begin=kb, k_end=ke, include_base=False)
        pref = O.fourier_llf(img.astype(np.float64), lev, K, 510.0, 20.0, 2.0, k_range=(kb, ke),
                             include_base=False)
        assert maxerr(part, pref) <= TOL_OUT
        parts.append(part)
    assert maxerr(sum(parts) + img, full) <= TOL_OUT
    base = gpu_run(F, img, lev, K, 510.0, 20.0, 2.0, k_begin=1, k_end=4, include_base=True)
    assert maxerr(base - parts[0], img) <= 1e-3


def test_batch_equals_frames(F):
    frames = np.stack([synth.uniform_image(40, 52, seed=50 + i) for i in range(3)])
    outb = gpu_run(F, frames, 4, 7, 510.0, 30.0, 3.0)
    for i in range(3):
        ref = O.fourier_llf(frames[i].astype(np.float64), 4, 7, 510.0, 30.0, 3.0)
        assert maxerr(outb[i], ref) <= TOL_OUT


@pytest.mark.parametrize("world", [1, 2, 3])
def test_gpu_partial_fn_channel_runs(F, world):
    """Config-3 order sharding through dist.gpu_partial_fn with batched channel
    runs (one plan per run of channels sharing an order range): the ranks'
    partials, summed as the NCCL reduce would, equal the full oracle per channel."""
    from paper_2206_04681_b200 import dist as D
    C, H, W, lev, K = 3, 40, 58, 4, 5
    rgb = np.stack([synth.uniform_image(H, W, seed=400 + c) for c in range(C)]).astype(np.float32)
    img = torch.from_numpy(rgb).cuda()
    total = torch.zeros((C, H, W), dtype=torch.float64)
    for segs in D.order_partition(C, K, world):
        fn = D.gpu_partial_fn(img, lev, K, 510.0, 20.0, 2.0)
        out = torch.zeros((C, H, W), device="cuda")
        for r in D.channel_runs(segs):
            fn(r, out[r.channel:r.channel + r.nch])
        torch.cuda.synchronize()
        total += out.cpu().double()
        for p in fn.plans.values():
            p.close()
    for c in range(C):
        ref = O.fourier_llf(rgb[c].astype(np.float64), lev, K, 510.0, 20.0, 2.0)
        assert maxerr(total[c].numpy(), ref) <= TOL_OUT


def test_filter_host_path(F):
    img = synth.config1_image(seed=1002)
    h_in = torch.from_numpy(img).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    with F.Plan(256, 256, 4, 4, 510.0, 30.0, 2.0) as p:
        F.fllf_filter_host(p.handle, h_in, h_out)
        torch.cuda.synchronize()
    ref = O.fourier_llf(img.astype(np.float64), 4, 4, 510.0, 30.0, 2.0)
    assert maxerr(h_out.numpy(), ref) <= TOL_OUT


@pytest.mark.parametrize("nb,batch", [(1, 1), (5, 1), (4, 2)])
def test_filter_host_frames_stream(F, nb, batch):
    """Streaming host path: nb batches through the double-buffered pipeline
    (odd counts end on either slot), each batch compared with the oracle;
    the in-pipeline L2 flush is switched on for one case."""
    H, W, lev, K = 45, 70, 4, 6
    frames = np.stack([synth.uniform_image(H, W, seed=300 + i) for i in range(nb * batch)]).astype(np.float32)
    h_in = torch.from_numpy(frames).pin_memory()
    h_out = torch.full_like(h_in, float("nan")).pin_memory()
    stride = batch * H * W * 4
    flush = torch.empty(1 << 20, device="cuda") if nb == 5 else None
    with F.Plan(H, W, lev, K, 510.0, 30.0, 3.0, batch=batch) as p:
        F.fllf_plan_set_l2_flush(p.handle, flush)
        F.fllf_filter_host_frames(p.handle, h_in, stride, h_out, stride, nb)
        torch.cuda.synchronize()
        with pytest.raises(F.FllfError):
            F.fllf_filter_host_frames(p.handle, h_in, stride, h_out, stride, -1)
    for i in range(nb * batch):
        ref = O.fourier_llf(frames[i].astype(np.float64), lev, K, 510.0, 30.0, 3.0)
        assert maxerr(h_out[i].numpy(), ref) <= TOL_OUT


def test_graph_cache_buffer_pairs(F):
    """fllf_filter keeps one CUDA graph per (input, output) buffer pair (4 cached,
    least recently used evicted): cycling 6 distinct pairs twice re-captures
    and replays correctly, each output equal to the first pair's result."""
    H, W = 37, 66
    img = synth.uniform_image(H, W, seed=77).astype(np.float32)
    ins = [torch.from_numpy(img).cuda() for _ in range(6)]
    outs = [torch.full((H, W), float("nan"), device="cuda") for _ in range(6)]
    with F.Plan(H, W, 3, 5, 510.0, 30.0, 2.0) as p:
        for _ in range(2):
            for a, b in zip(ins, outs):
                b.fill_(float("nan"))
                p.filter(a, b)
        torch.cuda.synchronize()
    ref = O.fourier_llf(img.astype(np.float64), 3, 5, 510.0, 30.0, 2.0)
    for b in outs:
        assert maxerr(b.cpu().numpy(), ref) <= TOL_OUT


def test_error_paths(F):
    with F.Plan(64, 64, 3, 4) as p:
        o = torch.empty((64, 64), device="cuda")
        with pytest.raises(F.FllfError) as e:
            p.apply(o)
        assert e.value.status == F.FLLF_ERR_NOT_BUILT
        narrow = torch.empty((64, 60), device="cuda")
        with pytest.raises(F.FllfError) as e:
            F.fllf_build_fourier_pyramids(p.handle, narrow)
        assert e.value.status == F.FLLF_ERR_BAD_POINTER
        p.build(torch.zeros((64, 64), device="cuda"))
        with pytest.raises(F.FllfError) as e:
            p.read_pyramid(0, 3, 0, torch.empty((8, 8), device="cuda"))
        assert e.value.status == F.FLLF_ERR_INVALID_ARGUMENT


# ---------------------------------------------------- BASELINE configs 2-5
def test_config2_full(F):
    c = synth.CONFIGS[2]
    img = synth.config2_image()
    ref = O.fourier_llf(img.astype(np.float64), c["levels"], c["K"], c["T"], c["sigma_r"], c["m"])
    out = gpu_run(F, img, c["levels"], c["K"], c["T"], c["sigma_r"], c["m"])
    assert maxerr(out, ref) <= TOL_OUT


def test_config3_rgb_full(F):
    c = synth.CONFIGS[3]
    rgb = synth.config3_rgb()
    out = gpu_run(F, rgb, c["levels"], c["K"], c["T"], c["sigma_r"], c["m"])  # channels as batch
    for ch in range(3):
        ref = O.fourier_llf(rgb[ch].astype(np.float64), c["levels"], c["K"], c["T"], c["sigma_r"], c["m"])
        assert maxerr(out[ch], ref) <= TOL_OUT, ch


@pytest.mark.parametrize("j", [0, 9])
def test_config4_maps_full(F, j):
    c = synth.CONFIGS[4]
    img = synth.config2_image(seed=4000, H=c["H"], W=c["W"])
    s, mm = synth.config4_maps(j)
    ref = O.fourier_llf(img.astype(np.float64), c["levels"], c["K"], c["T"],
                        sigma_map=s.astype(np.float64), m_map=mm.astype(np.float64))
    out = gpu_run(F, img, c["levels"], c["K"], c["T"], mode=F.FLLF_MAPS, smap=s, mmap=mm)
    assert maxerr(out, ref) <= TOL_OUT


def test_config5_batch_sampled(F):
    """All 64 frames run as one batched plan (the launch configuration of the
    config-5 bench); frames 0, 31, 63 are compared in full with the oracle."""
    c = synth.CONFIGS[5]
    frames = synth.config5_frames(64)
    out = gpu_run(F, frames, c["levels"], c["K"], c["T"], c["sigma_r"], c["m"])
    assert np.isfinite(out).all()
    for f in (0, 31, 63):
        ref = O.fourier_llf(frames[f].astype(np.float64), c["levels"], c["K"], c["T"], c["sigma_r"], c["m"])
        assert maxerr(out[f], ref) <= TOL_OUT, f
