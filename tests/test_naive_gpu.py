"""GPU parity of the naive-LLF ground truth (NEXT-2; Sec. II-C)
through the C ABI: against the fp64 oracle's brute-force naive LLF (exact
Gaussian remap and truncated-series remap) and against the exact identity
Fourier LLF(K) == naive LLF(r_K) with the GPU Fourier path itself."""
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


def gpu_naive(F, img, levels, K, T, sig, m, mode):
    H, W = img.shape
    d = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).cuda()
    out = torch.full_like(d, float("nan"))
    with F.Plan(H, W, levels, K, T, sig, m) as p:
        F.fllf_naive_llf(p.handle, d, out, mode)
        torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("shape,levels,sig,m", [((13, 10), 3, 30.0, 2.0), ((20, 17), 4, 20.0, 3.0),
                                                 ((33, 40), 5, 30.0, -1.0), ((7, 6), 2, 10.0, 4.0)])
def test_naive_exact_vs_oracle(F, shape, levels, sig, m):
    img = synth.uniform_image(*shape, seed=40 + levels)
    ref = O.naive_llf(img.astype(np.float64), levels, lambda I, g, l, q: O.remap_exact(I, g, sig, m))
    out = gpu_naive(F, img, levels, 4, 510.0, sig, m, F.REMAP_EXACT)
    assert np.abs(out - ref).max() <= TOL


@pytest.mark.parametrize("shape,levels,K,T", [((21, 14), 3, 4, 405.9), ((40, 31), 4, 6, 510.0)])
def test_naive_series_vs_oracle(F, shape, levels, K, T):
    img = synth.uniform_image(*shape, seed=K)
    c = O.fourier_coefficients(K, T, 30.0, 2.0)
    ref = O.naive_llf(img.astype(np.float64), levels, lambda I, g, l, q: O.remap_fourier(I, g, c["a"], c["omega"]))
    out = gpu_naive(F, img, levels, K, T, 30.0, 2.0, F.REMAP_SERIES)
    assert np.abs(out - ref).max() <= TOL


@pytest.mark.parametrize("K", [3, 8])
def test_identity_fourier_equals_naive_series_on_gpu(F, K):
    """Fourier LLF with K terms == naive LLF with r_K (exact identity), both on the GPU."""
    img = synth.config2_image(H=64, W=48)
    d = torch.from_numpy(img).cuda()
    four = torch.empty_like(d)
    with F.Plan(64, 48, 4, K, 510.0, 30.0, 3.0) as p:
        p.filter(d, four)
        torch.cuda.synchronize()
    naive = gpu_naive(F, img, 4, K, 510.0, 30.0, 3.0, F.REMAP_SERIES)
    assert np.abs(four.cpu().numpy() - naive).max() <= TOL


def test_naive_errors(F):
    d = torch.zeros((128, 128), dtype=torch.float32, device="cuda")
    with F.Plan(128, 128, 6, 4, 510.0, 30.0, 1.0) as p:   # too many levels for the naive tool
        with pytest.raises(F.FllfError):
            F.fllf_naive_llf(p.handle, d, d.clone(), F.REMAP_EXACT)
    with F.Plan(128, 128, 3, 4, 510.0, 30.0, 1.0, batch=2) as p:
        with pytest.raises(F.FllfError):
            F.fllf_naive_llf(p.handle, d, d.clone(), F.REMAP_EXACT)
