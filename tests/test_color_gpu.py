"""GPU parity of the NEXT-3 path (colour + variance-driven gain map, Sec. IV
P:373-377 with Sec. III-B per-pixel m) through the C ABI, against the fp64
oracle (oracle/color_gain.py).  Bar: the north star's 2e-3 max-abs on the
0-255 scale for the filtered RGB output; the intermediate planes get
tolerances derived from fp32 rounding."""
import numpy as np
import pytest
import torch
from scipy import ndimage

from oracle import color_gain as C

pytestmark = pytest.mark.gpu

TOL_OUT = 2e-3    # north star
TOL_YUV = 1e-4    # 3-term fp32 dot products of values <= 255
TOL_GAIN = 1e-5   # fp64 window sums; fp32 input and output rounding


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_04681_b200 import fllf
    return fllf


def rgb_image(H, W, seed):
    """Three correlated smooth-plus-texture channels in [0, 255] (config-3 style)."""
    rng = np.random.default_rng(seed)
    base = ndimage.gaussian_filter(rng.uniform(0, 1, (H, W)), 2.0, mode="mirror")
    out = []
    for c in range(3):
        e = ndimage.gaussian_filter(rng.uniform(0, 1, (H, W)), 1.0, mode="mirror")
        x = 0.8 * (base - base.mean()) / (base.std() + 1e-9) + 0.45 * (e - e.mean()) / (e.std() + 1e-9)
        out.append(np.clip(127.5 + 45.0 * x, 0, 255))
    return np.stack(out).astype(np.float32)


def test_yuv_roundtrip_and_oracle(F):
    rgb = rgb_image(37, 53, 1)
    d_rgb = torch.from_numpy(rgb).cuda()
    d_yuv = torch.empty_like(d_rgb)
    d_back = torch.empty_like(d_rgb)
    F.fllf_rgb_to_yuv(d_rgb, d_yuv)
    F.fllf_yuv_to_rgb(d_yuv, d_back)
    torch.cuda.synchronize()
    ref = C.rgb_to_yuv(rgb.astype(np.float64))
    assert np.abs(d_yuv.cpu().numpy() - ref).max() <= TOL_YUV
    assert np.abs(d_back.cpu().numpy() - rgb).max() <= TOL_YUV


@pytest.mark.parametrize("shape,r", [((64, 96), 3), ((9, 13), 12), ((33, 70), 0), ((130, 257), 7)])
def test_gain_map_vs_oracle(F, shape, r):
    rng = np.random.default_rng(r + shape[0])
    y = ndimage.gaussian_filter(rng.uniform(0, 255, shape), 1.2, mode="mirror").astype(np.float32)
    d_y = torch.from_numpy(y).cuda()
    d_m = torch.full(shape, float("nan"), dtype=torch.float32, device="cuda")
    F.fllf_gain_map(d_y, d_m, r, 0.5, 4.0, 150.0)
    torch.cuda.synchronize()
    ref = C.gain_map(y.astype(np.float64), r, 0.5, 4.0, 150.0)
    assert np.abs(d_m.cpu().numpy() - ref).max() <= TOL_GAIN * 4.0


@pytest.mark.parametrize("shape,levels,K,r", [((61, 90), 4, 8, 3), ((48, 33), 3, 5, 1), ((270, 480), 5, 12, 4)])
def test_enhance_rgb_vs_oracle(F, shape, levels, K, r):
    H, W = shape
    rgb = rgb_image(H, W, 7 + K)
    T, sig, m_lo, m_hi, v_ref = 510.0, 30.0, 0.5, 3.0, 120.0
    d_rgb = torch.from_numpy(rgb).cuda()
    d_out = torch.full_like(d_rgb, float("nan"))
    with F.Plan(H, W, levels, K, T, sig, 1.0) as p:
        F.fllf_enhance_rgb(p.handle, d_rgb, d_out, r, m_lo, m_hi, v_ref)
        torch.cuda.synchronize()
    ref = C.enhance_rgb(rgb.astype(np.float64), levels, K, T, sig, r, m_lo, m_hi, v_ref)
    assert np.abs(d_out.cpu().numpy() - ref).max() <= TOL_OUT


def test_enhance_rgb_errors(F):
    d = torch.zeros((3, 16, 16), dtype=torch.float32, device="cuda")
    o = torch.zeros_like(d)
    with F.Plan(16, 16, 3, 4, 510.0, 30.0, 1.0, batch=2) as p:
        with pytest.raises(F.FllfError):
            F.fllf_enhance_rgb(p.handle, d, o, 1, 0.5, 2.0, 100.0)
    with F.Plan(16, 16, 3, 4, 510.0, 30.0, 1.0) as p:
        with pytest.raises(F.FllfError):
            F.fllf_enhance_rgb(p.handle, d, o, 99, 0.5, 2.0, 100.0)   # radius too large
        with pytest.raises(F.FllfError):
            F.fllf_enhance_rgb(p.handle, d, o, 1, 0.5, 2.0, 0.0)                # v_ref <= 0
        with pytest.raises(F.FllfError):
            F.fllf_enhance_rgb(p.handle, d, d, 1, 0.5, 2.0, 100.0)              # aliasing
