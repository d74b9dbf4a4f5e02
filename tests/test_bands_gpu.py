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
