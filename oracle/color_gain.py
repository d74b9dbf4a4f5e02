"""Colour handling and the variance-driven gain map of the pixel-by-pixel
enhancement -- fp64 CPU ORACLE.

TEST INFRASTRUCTURE ONLY (same rules as ``fllf_oracle``): nothing on the
product path imports this module; it shares no code with the CUDA path.

What the paper says (Sec. IV):
  "The degree of enhancement is determined according to the variance of the
   pixels in a local window; the low variance is a small enhancement."
  "For color processing, LLF is applied to the Y channel of the YUV color
   space, and the other components are kept."
and Sec. III-B: the per-pixel parameters replace the coefficients
of Eq. 14 (``fllf_oracle.fourier_llf`` with ``sigma_map`` / ``m_map``).

Readings (R13-R16; the paper is silent on all four):
R13  YUV = BT.601 full range (the JPEG YCbCr matrix, chroma zero-centred, no
     offsets, no subsampling -- "the other components are kept").
R14  Local variance over the (2r+1)x(2r+1) window centred on the pixel,
     population form (divide by (2r+1)^2), reflect-101 borders (R2).
R15  Gain m_p = m_lo + (m_hi - m_lo) * min(1, v_p / v_ref): monotone in the
     variance, m_lo for flat regions ("low variance is a small enhancement").
R16  sigma_r stays uniform; only m varies per pixel ("we can also
     change the magnification factor of m to m_p").
"""
from __future__ import annotations

import numpy as np

from oracle import fllf_oracle as O

__all__ = ["YUV_FROM_RGB", "RGB_FROM_YUV", "rgb_to_yuv", "yuv_to_rgb", "local_variance", "gain_map",
           "enhance_rgb"]

# R13: BT.601 luma weights (Y = 0.299 R + 0.587 G + 0.114 B); Cb, Cr scaled so
# that their range is [-127.5, 127.5] for 8-bit input (JPEG / JFIF YCbCr).
YUV_FROM_RGB = np.array([
    [0.299, 0.587, 0.114],
    [-0.299 / 1.772, -0.587 / 1.772, 0.5],
    [0.5, -0.587 / 1.402, -0.114 / 1.402],
])
RGB_FROM_YUV = np.linalg.inv(YUV_FROM_RGB)


def rgb_to_yuv(rgb: np.ndarray) -> np.ndarray:
    """Planar (3, H, W) RGB -> planar (3, H, W) YUV (R13), a 3x3 matrix per pixel."""
    x = np.asarray(rgb, dtype=np.float64)
    return np.einsum("ij,jhw->ihw", YUV_FROM_RGB, x)


def yuv_to_rgb(yuv: np.ndarray) -> np.ndarray:
    """Inverse of ``rgb_to_yuv``."""
    x = np.asarray(yuv, dtype=np.float64)
    return np.einsum("ij,jhw->ihw", RGB_FROM_YUV, x)


def local_variance(y: np.ndarray, radius: int) -> np.ndarray:
    """R14: v_p = mean_w(y^2) - mean_w(y)^2 over the (2r+1)^2 window around p,
    reflect-101 borders; written as the plain double loop over window offsets
    (gathers through ``fllf_oracle.reflect101``)."""
    y = np.asarray(y, dtype=np.float64)
    H, W = y.shape
    n = (2 * radius + 1) ** 2
    s1 = np.zeros_like(y)
    s2 = np.zeros_like(y)
    rows = np.arange(H)
    cols = np.arange(W)
    for dy in range(-radius, radius + 1):
        ry = O.reflect101(rows + dy, H)
        for dx in range(-radius, radius + 1):
            rx = O.reflect101(cols + dx, W)
            v = y[np.ix_(ry, rx)]
            s1 += v
            s2 += v * v
    mean = s1 / n
    return s2 / n - mean * mean


def gain_map(y: np.ndarray, radius: int, m_lo: float, m_hi: float, v_ref: float) -> np.ndarray:
    """R15: m_p = m_lo + (m_hi - m_lo) min(1, v_p / v_ref)."""
    v = local_variance(y, radius)
    return m_lo + (m_hi - m_lo) * np.minimum(1.0, v / v_ref)


def enhance_rgb(rgb, levels, K, T, sigma_r, radius, m_lo, m_hi, v_ref):
    """The Fig. 5 pipeline: RGB -> YUV; gain map from the local
    variance of Y; Fourier LLF of Y with per-pixel m (Sec. III-B, uniform
    sigma_r, R16); U, V kept; back to RGB.  No clamping (R8)."""
    yuv = rgb_to_yuv(rgb)
    y = yuv[0]
    m = gain_map(y, radius, m_lo, m_hi, v_ref)
    s = np.full_like(y, float(sigma_r))
    yo = O.fourier_llf(y, levels, K, T, sigma_map=s, m_map=m)
    out = yuv.copy()
    out[0] = yo
    return yuv_to_rgb(out)
