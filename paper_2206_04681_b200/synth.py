"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the tests, ``bench.py`` and ``smoke()``; it holds
NONE of the method's arithmetic (no pyramid, remap or Fourier code) -- only
image synthesis.  Both the CUDA path and the oracle receive the same fp32
arrays produced here.

The paper's own test images (ten 512x512 8-bit grayscale photographs, P:297;
Lighthouse/Flower/Beach) are not available; these
generators stand in for them with the same value range [0, 255], grayscale
structure (smooth shading, strong step edges, piecewise-constant regions and
fine texture) and the sizes BASELINE.json's five configs name.  Recipe
("Input recipe"):

  rng     = numpy.random.Generator(PCG64(seed))
  smooth  = scipy.ndimage.gaussian_filter(x, s, mode="mirror", truncate=4)
  nrm(x)  = (x - min) / (max - min)
  seed    = 1000*config + frame (+100*channel, +10000*map index)

  config 1: 60 + 100 nrm(smooth(U[0,1), 3)) + 4 random step edges of height
            +-100, clipped to [0, 255]
  config 2: Voronoi partition (24 sites, levels U[30,225]) + 40 (nrm(smooth(U,3)) - .5)
            + 10 sin(2 pi (x cos phi + y sin phi)/lambda) per region
            (phi ~ U[0,pi), lambda ~ U[3,8] px), clipped
  config 3: X_c = 127.5 + sqrt(.8)(B - mean B) + sqrt(.2)(E_c - mean E_c), B, E_c
            config-2 fields -> inter-channel correlation ~0.8, clipped
  config 4: config-2 image; maps sigma_r = 10 + 50 nrm(S_j), m = .5 + 3.5 nrm(V_j)
            with S_j, V_j very smooth fields (smooth(U, 32) computed at 1/8
            resolution as smooth(U, 4) and bilinearly enlarged x8)
  config 5: 64 config-2 frames, seeds 5000..5063
"""
from __future__ import annotations

import numpy as np
from scipy import ndimage

__all__ = ["rng_for", "config1_image", "voronoi_texture_image", "config2_image",
           "config3_rgb", "config4_maps", "config5_frames", "uniform_image",
           "CONFIGS"]


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed)))


def _smooth(x, s):
    return ndimage.gaussian_filter(x, s, mode="mirror", truncate=4.0)


def _nrm(x):
    lo, hi = float(x.min()), float(x.max())
    return (x - lo) / (hi - lo) if hi > lo else np.zeros_like(x)


def uniform_image(H, W, seed, lo=0.0, hi=255.0) -> np.ndarray:
    """Plain U[lo,hi) noise (used for small ragged parity cases)."""
    return rng_for(seed).uniform(lo, hi, (H, W)).astype(np.float32)


def config1_image(seed: int = 1000, H: int = 256, W: int = 256) -> np.ndarray:
    rng = rng_for(seed)
    img = 60.0 + 100.0 * _nrm(_smooth(rng.random((H, W)), 3.0))
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    for _ in range(4):
        px = rng.uniform(0.1 * W, 0.9 * W)
        py = rng.uniform(0.1 * H, 0.9 * H)
        ang = rng.uniform(0.0, np.pi)
        sign = 1.0 if rng.random() < 0.5 else -1.0
        side = (xx - px) * np.sin(ang) - (yy - py) * np.cos(ang) > 0
        img = img + sign * 100.0 * side
    return np.clip(img, 0.0, 255.0).astype(np.float32)


def voronoi_texture_image(seed: int, H: int, W: int, sites: int = 24) -> np.ndarray:
    """Config-2 style field (float64, unclipped)."""
    rng = rng_for(seed)
    sy = rng.uniform(0, H, sites)
    sx = rng.uniform(0, W, sites)
    level = rng.uniform(30.0, 225.0, sites)
    phi = rng.uniform(0.0, np.pi, sites)
    lam = rng.uniform(3.0, 8.0, sites)
    noise = _smooth(rng.random((H, W)), 3.0)
    y = np.arange(H, dtype=np.float64)[:, None]
    x = np.arange(W, dtype=np.float64)[None, :]
    best = np.full((H, W), np.inf)
    region = np.zeros((H, W), dtype=np.int32)
    for s in range(sites):
        d = (y - sy[s]) ** 2 + (x - sx[s]) ** 2
        closer = d < best
        best = np.where(closer, d, best)
        region = np.where(closer, s, region)
    tex = 10.0 * np.sin(2.0 * np.pi * (x * np.cos(phi[region]) + y * np.sin(phi[region]))
                        / lam[region])
    return level[region] + 40.0 * (_nrm(noise) - 0.5) + tex


def config2_image(seed: int = 2000, H: int = 1080, W: int = 1920) -> np.ndarray:
    return np.clip(voronoi_texture_image(seed, H, W), 0.0, 255.0).astype(np.float32)


def config3_rgb(seed: int = 3000, H: int = 2160, W: int = 3840) -> np.ndarray:
    """(3, H, W) fp32; channel c uses base field B (seed) and E_c (seed + 100*(c+1))."""
    B = voronoi_texture_image(seed, H, W)
    out = []
    for c in range(3):
        E = voronoi_texture_image(seed + 100 * (c + 1), H, W)
        X = 127.5 + np.sqrt(0.8) * (B - B.mean()) + np.sqrt(0.2) * (E - E.mean())
        out.append(np.clip(X, 0.0, 255.0))
    return np.stack(out).astype(np.float32)


def _very_smooth(rng, H, W):
    h, w = (H + 7) // 8, (W + 7) // 8
    f = _smooth(rng.random((h, w)), 4.0)
    big = ndimage.zoom(f, (H / h, W / w), order=1, mode="nearest", grid_mode=True)
    return big[:H, :W]


def config4_maps(j: int, seed: int = 4000, H: int = 2160, W: int = 3840):
    """Parameter-map pair j (0..9): sigma_r in [10, 60], m in [0.5, 4]."""
    rng = rng_for(seed + 10000 * (j + 1))
    sig = 10.0 + 50.0 * _nrm(_very_smooth(rng, H, W))
    m = 0.5 + 3.5 * _nrm(_very_smooth(rng, H, W))
    return sig.astype(np.float32), m.astype(np.float32)


def config5_frames(n: int = 64, H: int = 1080, W: int = 1920, first: int = 0) -> np.ndarray:
    return np.stack([config2_image(5000 + f, H, W) for f in range(first, first + n)])


# The five BASELINE.json configs (levels, K, T, sigma_r, m).  T = 255*2 for all
# (config 1 states it; the others do not, reading R10).
CONFIGS = {
    1: dict(H=256, W=256, levels=4, K=4, T=510.0, sigma_r=30.0, m=2.0),
    2: dict(H=1080, W=1920, levels=6, K=8, T=510.0, sigma_r=30.0, m=3.0),
    3: dict(H=2160, W=3840, levels=7, K=10, T=510.0, sigma_r=20.0, m=2.0, channels=3),
    4: dict(H=2160, W=3840, levels=7, K=12, T=510.0, maps=10),
    5: dict(H=1080, W=1920, levels=6, K=16, T=510.0, sigma_r=30.0, m=3.0, frames=64),
}
