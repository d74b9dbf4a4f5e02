"""Pins of the NEXT-3 oracle (oracle/color_gain.py): BT.601 YUV, local variance,
variance-driven gain map and the colour pipeline, against textbook values,
closed forms, library routines and reductions -- none re-types the oracle."""
import json
import os

import numpy as np
import pytest
from scipy import ndimage

from oracle import color_gain as C
from oracle import fllf_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bt601_full_range.json")))


def test_yuv_matrix_textbook_values():
    """R13: the JFIF / ITU-T T.871 full-range YCbCr coefficients (golden file)."""
    np.testing.assert_allclose(C.YUV_FROM_RGB, np.array(GOLD["ycbcr_from_rgb"]), atol=5e-7)
    np.testing.assert_allclose(C.RGB_FROM_YUV, np.array(GOLD["rgb_from_ycbcr"]), atol=5e-7)


def test_yuv_gray_and_roundtrip():
    rng = np.random.default_rng(3)
    g = rng.uniform(0, 255, (5, 7))
    yuv = C.rgb_to_yuv(np.stack([g, g, g]))
    np.testing.assert_allclose(yuv[0], g, atol=1e-12)
    np.testing.assert_allclose(yuv[1:], 0.0, atol=1e-12)
    rgb = rng.uniform(0, 255, (3, 9, 4))
    np.testing.assert_allclose(C.yuv_to_rgb(C.rgb_to_yuv(rgb)), rgb, atol=1e-10)


def _brute_variance(y, r):
    H, W = y.shape
    out = np.empty_like(y)
    for i in range(H):
        for j in range(W):
            win = [y[O.reflect101(i + a, H), O.reflect101(j + b, W)]
                   for a in range(-r, r + 1) for b in range(-r, r + 1)]
            out[i, j] = np.var(np.array(win, dtype=np.float64))
    return out


@pytest.mark.parametrize("shape,r", [((9, 13), 1), ((7, 5), 2), ((12, 12), 3)])
def test_local_variance_brute_force_and_scipy(shape, r):
    rng = np.random.default_rng(sum(shape) + r)
    y = rng.uniform(0, 255, shape)
    v = C.local_variance(y, r)
    np.testing.assert_allclose(v, _brute_variance(y, r), rtol=1e-10, atol=1e-8)
    # library path: box means with scipy's "mirror" (= reflect-101) borders
    m1 = ndimage.uniform_filter(y, size=2 * r + 1, mode="mirror")
    m2 = ndimage.uniform_filter(y * y, size=2 * r + 1, mode="mirror")
    np.testing.assert_allclose(v, m2 - m1 * m1, rtol=1e-9, atol=1e-7)


def test_local_variance_closed_forms():
    assert np.abs(C.local_variance(np.full((6, 8), 37.5), 2)).max() < 1e-9
    # interior of a 0/255 checkerboard, r = 1: 5 of one value and 4 of the other
    y = (np.indices((9, 9)).sum(0) % 2) * 255.0
    v = C.local_variance(y, 1)
    expect = 255.0 ** 2 * (5 / 9) * (4 / 9)
    np.testing.assert_allclose(v[2:-2, 2:-2], expect, rtol=1e-12)


def test_gain_map_ramp():
    y = np.zeros((8, 8))
    y[:, 4:] = 100.0  # a vertical step: variance > 0 only near the edge
    g = C.gain_map(y, 1, 0.5, 4.0, 1000.0)
    assert np.all(g[:, :2] == 0.5) and np.all(g[:, -2:] == 0.5)     # flat -> m_lo
    v = C.local_variance(y, 1)
    edge = v > 0
    np.testing.assert_allclose(g[edge], 0.5 + 3.5 * np.minimum(1, v[edge] / 1000.0))
    assert C.gain_map(y, 1, 0.5, 4.0, 1.0)[edge].min() == 4.0       # saturated -> m_hi


def test_enhance_rgb_reductions():
    rng = np.random.default_rng(11)
    gray = ndimage.gaussian_filter(rng.uniform(0, 255, (20, 23)), 1.5, mode="mirror")
    rgb = np.stack([gray, gray, gray])
    # constant gain (m_lo == m_hi): the scalar Fourier LLF of the luma, gray stays gray
    out = C.enhance_rgb(rgb, 3, 6, 510.0, 30.0, 2, 2.0, 2.0, 100.0)
    ref = O.fourier_llf(gray, 3, 6, 510.0, 30.0, 2.0)
    for c in range(3):
        np.testing.assert_allclose(out[c], ref, atol=1e-9)
    # zero gain: identity
    rgb2 = rng.uniform(0, 255, (3, 11, 10))
    np.testing.assert_allclose(C.enhance_rgb(rgb2, 3, 4, 510.0, 30.0, 1, 0.0, 0.0, 100.0), rgb2, atol=1e-9)
