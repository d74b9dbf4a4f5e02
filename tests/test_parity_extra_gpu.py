"""More GPU parity cases for kernel variants added in round 1: the Clenshaw
MAPS path (16-byte aligned maps, W % 4 == 0) vs its forward-recurrence
fallback, K at FLLF_MAX_K, odd order counts in COEFFS mode, large sigma*K
(per-order coefficients underflowing to 0) and a caller image whose rows are
not 16-byte aligned (no TMA for the level-0 header).  Bar: 2e-3 (north star)."""
import numpy as np
import pytest
import torch

from oracle import fllf_oracle as O
from paper_2206_04681_b200 import synth

pytestmark = pytest.mark.gpu
TOL = 2e-3


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_04681_b200 import fllf
    return fllf


def maps_case(F, H, W, levels, K, s, mm, offset=0):
    img = synth.uniform_image(H, W, seed=H + K)
    d = torch.from_numpy(img).cuda()
    out = torch.full_like(d, float("nan"))
    if offset:  # maps as column-offset views: 4-byte aligned rows only (forward-kernel fallback)
        sb = torch.zeros((H, W + offset), device="cuda")
        mb = torch.zeros((H, W + offset), device="cuda")
        sb[:, offset:] = torch.from_numpy(s).cuda()
        mb[:, offset:] = torch.from_numpy(mm).cuda()
        ds, dm = sb[:, offset:], mb[:, offset:]
    else:
        ds, dm = torch.from_numpy(s).cuda(), torch.from_numpy(mm).cuda()
    with F.Plan(H, W, levels, K, 510.0, 30.0, 1.0) as p:
        p.build(d)
        p.apply(out, mode=F.FLLF_MAPS, sigma_map=ds, m_map=dm)
        torch.cuda.synchronize()
    ref = O.fourier_llf(img.astype(np.float64), levels, K, 510.0, sigma_map=s.astype(np.float64),
                        m_map=mm.astype(np.float64))
    return float(np.abs(out.cpu().numpy() - ref).max())


@pytest.mark.parametrize("H,W,levels,K,offset", [(90, 132, 5, 12, 0), (121, 64, 4, 7, 0), (90, 132, 5, 12, 1),
                                                  (67, 200, 3, 3, 0)])
def test_maps_clenshaw_and_fallback(F, H, W, levels, K, offset):
    rng = np.random.default_rng(H * W)
    s = rng.uniform(10.0, 60.0, (H, W)).astype(np.float32)
    mm = rng.uniform(-1.0, 4.0, (H, W)).astype(np.float32)
    assert maps_case(F, H, W, levels, K, s, mm, offset) <= TOL


def test_maps_large_sigma_k(F):
    """sigma_r = 60, K = 32: e^{-k^2 beta} underflows for the top orders (a_k -> 0)."""
    H, W = 48, 64
    s = np.full((H, W), 60.0, np.float32)
    s[:, 32:] = 55.0
    mm = np.full((H, W), 3.0, np.float32)
    assert maps_case(F, H, W, 3, 32, s, mm) <= TOL


@pytest.mark.parametrize("K", [32, 7])
def test_max_and_odd_orders_coeffs(F, K):
    img = synth.uniform_image(57, 96, seed=K)
    a = O.fourier_coefficients(K, 510.0, 25.0, 2.5)["a"]
    ref = O.fourier_llf(img.astype(np.float64), 4, K, 510.0, a=a)
    d = torch.from_numpy(img).cuda()
    out = torch.full_like(d, float("nan"))
    with F.Plan(57, 96, 4, K, 510.0, 25.0, 2.5) as p:
        p.build(d)
        p.apply(out, mode=F.FLLF_COEFFS, a_k=a)
        torch.cuda.synchronize()
    assert float(np.abs(out.cpu().numpy() - ref).max()) <= TOL


def test_unaligned_caller_image(F):
    """Image rows at a 4-byte (not 16-byte) aligned pitch and base: the level-0
    header falls back to direct loads."""
    H, W = 70, 128
    img = synth.uniform_image(H, W, seed=77)
    buf = torch.zeros((H * (W + 1) + 1,), device="cuda")
    view = buf[1:1 + H * (W + 1)].view(H, W + 1)[:, :W]
    view.copy_(torch.from_numpy(img).cuda())
    out = torch.full((H, W), float("nan"), device="cuda")
    with F.Plan(H, W, 4, 8, 510.0, 30.0, 3.0) as p:
        p.filter(view, out)
        torch.cuda.synchronize()
    ref = O.fourier_llf(img.astype(np.float64), 4, 8, 510.0, 30.0, 3.0)
    assert float(np.abs(out.cpu().numpy() - ref).max()) <= TOL
