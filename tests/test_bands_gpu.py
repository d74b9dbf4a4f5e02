"""NEXT-1 row bands on one GPU: P bands of a frame, run level by level with the
halo rows exchanged between the bands' stored rows (the single-process
emulation of the multi-GPU band_filter: no kernel waits on another), must
reproduce the whole-frame filter; and the whole frame must still match the
fp64 oracle.  Bar: 2e-3 vs the oracle (north star); band vs whole frame:
identical arithmetic on identical inputs -> 1e-5."""
import numpy as np
import pytest
import torch

from oracle import fllf_oracle as O
from paper_2206_04681_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_04681_b200 import fllf
    return fllf


@pytest.mark.parametrize("H,W,levels,K,P", [(256, 200, 4, 6, 2), (300, 173, 5, 8, 3), (1080, 480, 6, 8, 4),
                                             (517, 96, 3, 5, 7)])
def test_bands_match_whole_frame(F, H, W, levels, K, P):
    from paper_2206_04681_b200 import dist as D
    img = torch.from_numpy(synth.config2_image(seed=H + P, H=H, W=W)).cuda()
    full = torch.empty_like(img)
    with F.Plan(H, W, levels, K, 510.0, 30.0, 3.0) as p:
        p.filter(img, full)
    out = torch.full_like(img, float("nan"))
    bands = [D.GpuBand(H, W, levels, K, 510.0, 30.0, 3.0, b) for b in D.band_partition(H, levels, P)]
    try:
        D.band_filter_local(bands, img, out)
        torch.cuda.synchronize()
    finally:
        for b in bands:
            b.close()
    assert torch.isfinite(out).all()
    assert float((out - full).abs().max()) <= 1e-5
    if H * W <= 300 * 173:
        ref = O.fourier_llf(img.cpu().numpy().astype(np.float64), levels, K, 510.0, 30.0, 3.0)
        assert np.abs(out.cpu().numpy() - ref).max() <= 2e-3


def test_band_plan_errors(F):
    with pytest.raises(F.FllfError):   # boundary not a multiple of 2^(levels-1)
        F.Plan(256, 64, 4, 4, row_begin=4, row_end=256)
    with pytest.raises(F.FllfError):   # bands need batch 1
        F.Plan(256, 64, 4, 4, batch=2, row_begin=0, row_end=128)
    with F.Plan(256, 64, 4, 4, row_begin=0, row_end=128) as p:
        d = torch.zeros((128, 64), device="cuda")
        with pytest.raises(F.FllfError):
            p.apply(d, mode=F.FLLF_MAPS, sigma_map=d, m_map=d)


@pytest.mark.parametrize("H,W,levels,K,P", [(2160, 3840, 7, 10, 2), (1080, 480, 6, 8, 4)])
def test_bands_own_buffers(F, H, W, levels, K, P):
    """Each band holds only its rows (+ the 2 halo rows above / below) in a
    buffer of its own, as a rank of the multi-GPU band_filter does: the plan's
    row-0 image pointer then lies below the allocation, and every TMA tensor
    map must still cover only the rows the band reads / stores (DESIGN.md
    section 11: such maps faulted before they were restricted)."""
    from paper_2206_04681_b200 import dist as D
    img = torch.from_numpy(synth.config2_image(seed=H + W + P, H=H, W=W)).cuda()
    full = torch.empty_like(img)
    with F.Plan(H, W, levels, K, 510.0, 30.0, 3.0) as p:
        p.filter(img, full)
    bands = [D.GpuBand(H, W, levels, K, 510.0, 30.0, 3.0, b) for b in D.band_partition(H, levels, P)]
    try:
        ins, outs = [], []
        for gb in bands:
            rb, re_ = gb.band
            lo, hi = max(0, rb - 2), min(H, re_ + 2)
            ins.append((img[lo:hi].clone(), rb - lo))
            outs.append(torch.full((re_ - rb, W), float("nan"), device="cuda"))
        torch.cuda.synchronize()
        pitch = W * 4
        for step in D.band_schedule(levels):
            if step[0] == "xchg":
                l = step[1]
                for kind in step[2]:
                    views = [gb.view(l, kind) for gb in bands]
                    for i in range(len(bands) - 1):
                        (vu, fu), (vd, fd) = views[i], views[i + 1]
                        _, bot_u, _, send_dn_u, _, _ = D.halo_slices(fu, vu.shape[1], bands[i].own(l))
                        top_d, _, send_up_d, _, _, _ = D.halo_slices(fd, vd.shape[1], bands[i + 1].own(l))
                        vu[:, bot_u] = vd[:, send_up_d]
                        vd[:, top_d] = vu[:, send_dn_u]
            else:
                for gb, (ib, top), ob in zip(bands, ins, outs):
                    gb.run_step(step, ib.data_ptr() + top * pitch, pitch, ob.data_ptr(), pitch)
        torch.cuda.synchronize()
    finally:
        for b in bands:
            b.close()
    out = torch.cat(outs)
    assert torch.isfinite(out).all()
    assert float((out - full).abs().max()) <= 1e-5
