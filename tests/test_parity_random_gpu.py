"""Seeded random sweep of the whole path against the fp64 oracle: frame sizes
from the smallest a level count allows (coarsest level >= 3x3) to a few
tiles, ragged in both directions, 2..6 levels, K = 1..16, both T of the
paper, sigma_r 10..60, m of either sign, batches 1..3, with and without a
padded caller pitch, and all three apply modes (SCALAR through fllf_filter /
build + apply, COEFFS with a random odd remap, MAPS).  Bar: the north star's
2e-3 on the 0-255 scale."""
import numpy as np
import pytest
import torch

from oracle import fllf_oracle as O
from paper_2206_04681_b200 import synth

from test_parity_gpu import TOL_OUT, gpu_run, maxerr  # noqa: F401  (fixture F below)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_04681_b200 import fllf
    return fllf


def _case(seed):
    rng = np.random.default_rng(seed)
    levels = int(rng.integers(2, 7))
    lo = 3 << (levels - 1)  # smallest size whose coarsest level is >= 3 (ceil-halving)
    H = int(rng.integers(lo - (1 << (levels - 1)) + 1, lo + 160))
    W = int(rng.integers(lo - (1 << (levels - 1)) + 1, lo + 300))
    K = int(rng.integers(1, 17))
    T = float(rng.choice([405.9, 510.0]))
    sig = float(rng.uniform(10.0, 60.0))
    m = float(rng.choice([-1.0, 1.0]) * rng.uniform(0.2, 4.0))
    B = int(rng.integers(1, 4))
    pad = int(rng.choice([0, 0, 3]))
    mode = int(rng.integers(0, 3))
    return levels, H, W, K, T, sig, m, B, pad, mode, rng


def _fits(H, W, levels):
    h, w = H, W
    for _ in range(levels - 1):
        h, w = (h + 1) // 2, (w + 1) // 2
    return h >= 3 and w >= 3


@pytest.mark.parametrize("seed", range(96))
def test_random_config(F, seed):
    levels, H, W, K, T, sig, m, B, pad, mode, rng = _case(1000 + seed)
    if not _fits(H, W, levels):
        H, W = H + (1 << levels), W + (1 << levels)
    assert _fits(H, W, levels)
    frames = np.stack([synth.uniform_image(H, W, seed=5000 + 10 * seed + b) for b in range(B)]).astype(np.float32)
    if mode == 0:  # SCALAR
        out = gpu_run(F, frames, levels, K, T, sig, m, pitch_pad=pad)
        refs = [O.fourier_llf(f.astype(np.float64), levels, K, T, sig, m) for f in frames]
    elif mode == 1:  # COEFFS: any odd remap detail with period T
        a = rng.normal(0.0, 5.0, K) / (1.0 + np.arange(K))
        out = gpu_run(F, frames, levels, K, T, sig, m, mode=F.FLLF_COEFFS, a_k=a, pitch_pad=pad)
        refs = [O.fourier_llf(f.astype(np.float64), levels, K, T, a=a) for f in frames]
    else:  # MAPS: smooth sigma_r / m maps shared by the batch
        yy, xx = np.meshgrid(np.linspace(0, 1, H), np.linspace(0, 1, W), indexing="ij")
        smap = (10.0 + 40.0 * (0.5 + 0.5 * np.sin(3 * xx + 2 * yy))).astype(np.float32)
        mmap = (m * (0.5 + yy)).astype(np.float32)
        out = gpu_run(F, frames, levels, K, T, sig, m, mode=F.FLLF_MAPS, smap=smap, mmap=mmap, pitch_pad=pad)
        refs = [O.fourier_llf(f.astype(np.float64), levels, K, T, sigma_map=smap.astype(np.float64),
                              m_map=mmap.astype(np.float64)) for f in frames]
    out = out if out.ndim == 3 else out[None]
    for b in range(B):
        assert maxerr(out[b], refs[b]) <= TOL_OUT, (levels, H, W, K, T, sig, m, B, pad, mode)
