"""Pins for the fp64 oracle (CPU, -m "not gpu").

Each test checks the oracle against something OTHER than itself: values the
paper prints, hand evaluations, a library routine for a special case, closed
forms (Poisson summation, the linear-remap / Eq. 3 special case), exact
identities (Fourier LLF == naive LLF run with the truncated remap), invariants
and brute force on tiny inputs.  Citations "P:n" are PAPER.md lines.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import ndimage

from oracle import fllf_oracle as O
from fllf_testutil import GOLDEN

pytestmark = pytest.mark.filterwarnings("ignore")


def _rand(shape, seed, lo=0.0, hi=255.0):
    return np.random.default_rng(seed).uniform(lo, hi, shape)


# ---------------------------------------------------------------- pyramid ops
def test_border_hand_values():
    d = json.load(open(os.path.join(GOLDEN, "border_hand_values.json")))
    for c in d["cases"]:
        x = np.array(c["x"], dtype=np.float64)
        got = O.down(x) if c["op"] == "down" else O.up(x, c["n"])
        np.testing.assert_allclose(got, c["expect"], rtol=0, atol=1e-15, err_msg=c["hand"])


@pytest.mark.parametrize("shape", [(37, 23), (16, 16), (9, 14), (5, 6)])
def test_down_up_match_scipy_mirror(shape):
    """Special case reducing to a library routine: reflect-101 == scipy's
    ``mode='mirror'`` (d c b | a b c d | c b a).  down = correlate with the
    binomial then keep even samples; up = zero insertion then correlate with
    2x the binomial (readings R2, R5)."""
    w = np.array([1, 4, 6, 4, 1], dtype=np.float64) / 16.0
    x = _rand(shape, 1)
    ref = ndimage.correlate1d(ndimage.correlate1d(x, w, axis=1, mode="mirror"),
                              w, axis=0, mode="mirror")[::2, ::2]
    np.testing.assert_allclose(O.down(x), ref, rtol=0, atol=1e-12)
    c = _rand(((shape[0] + 1) // 2, (shape[1] + 1) // 2), 2)
    z = np.zeros(shape)
    z[::2, ::2] = c
    ref_up = ndimage.correlate1d(ndimage.correlate1d(z, 2 * w, axis=1, mode="mirror"),
                                 2 * w, axis=0, mode="mirror")
    np.testing.assert_allclose(O.up(c, shape), ref_up, rtol=0, atol=1e-12)


@pytest.mark.parametrize("shape,levels", [((37, 23), 4), ((64, 64), 5), ((13, 10), 3), ((1, 7), 3)])
def test_reconstruction(shape, levels):
    """Telescoping identity of Eq. 2 + Eq. 4: collapse(L[I]) == I."""
    I = _rand(shape, 3)
    assert np.abs(O.collapse(O.laplacian_pyramid(I, levels)) - I).max() <= 1e-9


def test_level_shapes_ceil_halving():
    assert O.level_shapes((1080, 1920), 6)[-1] == (34, 60)
    assert O.level_shapes((2160, 3840), 7)[-2:] == [(68, 120), (34, 60)]
    assert [s[0] for s in O.level_shapes((135, 17), 4)] == [135, 68, 34, 17]


# --------------------------------------------------------------- coefficients
def test_coefficients_paper_setting():
    g = json.load(open(os.path.join(GOLDEN, "coefficients_T405.9_sigma30.json")))
    c = O.fourier_coefficients(10, g["T"], g["sigma_r"], 1.0)
    assert abs(c["omega"][0] - g["omega_1"]) < g["abs_tol"]
    assert abs(c["alpha0"] - g["alpha_0"]) < g["abs_tol"]
    assert abs(c["alpha"][0] - g["alpha_1"]) < g["abs_tol"]
    assert abs(c["alpha_tilde"][0] - g["alpha_tilde_1"]) < g["abs_tol"]


def _detail(x, sigma, m):
    return m * x * np.exp(-x * x / (2 * sigma * sigma))


@pytest.mark.parametrize("K,T,sigma,m", [(4, 510.0, 30.0, 2.0), (8, 510.0, 30.0, 3.0),
                                         (10, 510.0, 20.0, 2.0), (12, 510.0, 10.0, 4.0),
                                         (12, 510.0, 60.0, 4.0), (16, 510.0, 30.0, 3.0),
                                         (10, 405.9, 30.0, 7.0)])
def test_series_poisson_identity(K, T, sigma, m):
    """Closed form for the truncation error.  a_k = (2/T) int d(x) sin(w_k x) dx
    over R (Eq. 9-11 with d(x) = m x exp(-x^2/2 sigma^2)), so by Poisson
    summation sum_{k>=1} a_k sin(w_k x) = sum_n d(x + nT) EXACTLY, hence
      S_K(x) - d(x) = sum_{n != 0} d(x + nT) - sum_{k > K} a_k sin(w_k x).
    A dropped factor 2, a wrong sqrt(2 pi)/T or a wrong omega breaks it."""
    x = np.linspace(-255.0, 255.0, 2041)
    cK = O.fourier_coefficients(K, T, sigma, m)
    SK = (cK["a"][:, None] * np.sin(cK["omega"][:, None] * x[None, :])).sum(0)
    Kbig = K + 200
    cB = O.fourier_coefficients(Kbig, T, sigma, m)
    tail = (cB["a"][K:, None] * np.sin(cB["omega"][K:, None] * x[None, :])).sum(0)
    alias = sum(_detail(x + n * T, sigma, m) for n in range(-6, 7) if n != 0)
    np.testing.assert_allclose(SK - _detail(x, sigma, m), alias - tail, rtol=0, atol=1e-9)
    # and the truncation error is within the bound expected for K
    bound = np.abs(cB["a"][K:]).sum() + np.abs(alias).max()
    assert np.abs(SK - _detail(x, sigma, m)).max() <= bound + 1e-12


def test_remap_exact_hand_value_and_sign():
    """r(100, 50) with m=1, sigma=30 (R1, enhancing sign):
    100 + 50 exp(-2500/1800) = 112.46761...; m>0 moves i AWAY from g."""
    v = O.remap_exact(100.0, 50.0, 30.0, 1.0)
    assert abs(v - (100.0 + 50.0 * math.exp(-2500.0 / 1800.0))) < 1e-12
    assert abs(v - 112.46761) < 1e-5
    assert O.remap_exact(40.0, 50.0, 30.0, 2.0) < 40.0


def test_period_eq12_matches_paper():
    g = json.load(open(os.path.join(GOLDEN, "period_eq12.json")))
    T = O.optimal_period(g["K"], g["sigma_r"], g["R"])
    assert abs(T - g["paper_T"]) < g["abs_tol"]
    # interior minimum and monotone in K (first erfc term grows with 2K+1)
    Ts = [O.optimal_period(k, 30.0, 256) for k in range(2, 16)]
    assert all(b >= a for a, b in zip(Ts, Ts[1:]))


# -------------------------------------------------------------- Fourier LLF
@pytest.mark.parametrize("shape,levels", [((13, 10), 3), ((9, 14), 4)])
@pytest.mark.parametrize("K", [3, 4, 8])
@pytest.mark.parametrize("T", [405.9, 510.0])
@pytest.mark.parametrize("m", [-1.0, 2.0, 3.0])
def test_fourier_equals_naive_with_truncated_remap(shape, levels, K, T, m):
    """Exact identity: Fourier LLF with K terms == naive LLF (brute
    force over every pixel and level) run with r_K(i,g) = i + sum a_k sin(w_k(i-g)),
    because every pyramid operator is linear.  Catches sign, index, level and
    up/down-pairing mistakes in the Eq. 14 assembly."""
    I = _rand(shape, 11)
    c = O.fourier_coefficients(K, T, 30.0, m)
    F = O.fourier_llf(I, levels, K, T, 30.0, m)
    N = O.naive_llf(I, levels, lambda A, g, l, q: O.remap_fourier(A, g, c["a"], c["omega"]))
    assert np.abs(F - N).max() <= 1e-10


def _step_smooth_32():
    rng = np.random.default_rng(7)
    I = 60 + 100 * ndimage.gaussian_filter(rng.random((32, 32)), 2.0, mode="mirror")
    I[:, 16:] += 80.0
    I[20:, :] -= 30.0
    return I


def test_convergence_to_exact_naive():
    """Fourier LLF -> naive LLF with the exact remap as K grows (north star).
    Rigorous bound: |L_l[X]| <= 2 sup|X| and collapse adds l_max detail
    levels, so |F_K - naive| <= 2 l_max e_K with e_K the series error."""
    I = _step_smooth_32()
    levels, T, sig, m = 4, 510.0, 30.0, 2.0
    N = O.naive_llf(I, levels, lambda A, g, l, q: O.remap_exact(A, g, sig, m))
    x = np.linspace(-255.0, 255.0, 5101)
    errs = []
    for K in (2, 4, 6, 8, 12, 16):
        F = O.fourier_llf(I, levels, K, T, sig, m)
        c = O.fourier_coefficients(K, T, sig, m)
        eK = np.abs((c["a"][:, None] * np.sin(c["omega"][:, None] * x)).sum(0)
                    - _detail(x, sig, m)).max()
        err = np.abs(F - N).max()
        assert err <= 2 * (levels - 1) * eK * 1.001 + 1e-9, (K, err, eK)
        errs.append(err)
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-5


def test_naive_linear_remap_is_pyramid_enhancement():
    """Textbook special case (Eq. 3): with the linear remap
    r(i,g) = i + beta (i - g), L_l[r(I,g_p)]_p = (1+beta) L_l[I]_p because
    L_l of a constant is 0; so naive LLF == collapse((1+beta) L_l, G_lmax)."""
    I = _rand((11, 13), 5)
    beta = 0.7
    N = O.naive_llf(I, 3, lambda A, g, l, q: A + beta * (A - g))
    L = O.laplacian_pyramid(I, 3)
    ref = O.collapse([(1 + beta) * L[0], (1 + beta) * L[1], L[2]])
    assert np.abs(N - ref).max() <= 1e-10


@pytest.mark.parametrize("K,expect_gamma", [(4, 0.572401), (16, 1.0)])
def test_small_range_gain(K, expect_gamma):
    """For I = c + eps P the remap is linear around g with slope
    1 + m gamma_K, gamma_K = sum_k alpha~_k omega_k (d/dx of the series at 0),
    so O = collapse((1 + m gamma_K) L_l[I] for l < l_max; G_lmax) + O(eps^3).
    Pins the enhancing sign (m > 0 => gain > 1).  gamma_16 = 1 - 3.5e-8."""
    T, sig, m = 510.0, 30.0, 2.0
    c = O.fourier_coefficients(K, T, sig, 1.0)
    gamma = float((c["alpha_tilde"] * c["omega"]).sum())
    assert abs(gamma - expect_gamma) < 1e-6
    eps = 1e-3
    I = 120.0 + eps * _rand((19, 17), 9, -1, 1)
    F = O.fourier_llf(I, 4, K, T, sig, m)
    L = O.laplacian_pyramid(I, 4)
    ref = O.collapse([(1 + m * gamma) * x for x in L[:-1]] + [L[-1]])
    assert np.abs(F - ref).max() <= 1e-9 * eps + 1e-11
    assert 1 + m * gamma > 1


def test_identity_cases():
    I = _rand((21, 18), 4)
    assert np.abs(O.fourier_llf(I, 4, 8, 510.0, 30.0, 0.0) - I).max() <= 1e-9
    C = np.full((21, 18), 77.25)
    assert np.abs(O.fourier_llf(C, 4, 8, 510.0, 30.0, 3.0) - C).max() <= 1e-9
    assert np.abs(O.naive_llf(C[:7, :6], 3, lambda A, g, l, q: O.remap_exact(A, g, 30.0, 3.0))
                  - C[:7, :6]).max() <= 1e-9


def test_invariants_shift_reflection_linearity():
    """Exact at any K: r_K(i+c, g+c) = r_K(i,g) + c and r_K(-i,-g) = -r_K(i,g),
    hence F(I+c) = F(I)+c and F(255-I) = 255-F(I); F is affine in m."""
    I = _rand((23, 29), 6)
    args = (4, 8, 510.0, 30.0)
    F = O.fourier_llf(I, *args, 2.0)
    assert np.abs(O.fourier_llf(I + 13.5, *args, 2.0) - (F + 13.5)).max() <= 1e-9
    assert np.abs(O.fourier_llf(255.0 - I, *args, 2.0) - (255.0 - F)).max() <= 1e-9
    F3 = O.fourier_llf(I, *args, 6.0)
    assert np.abs((F3 - I) - 3 * (F - I)).max() <= 1e-9


def test_level0_general_form_reduces_to_eq14_l0():
    """at l = 0 the same-level Fourier term vanishes, so
    L_0[O] = I - G_1 up + sum a_k (sin(w I) C~_1 up - cos(w I) S~_1 up)."""
    I = _rand((17, 12), 8)
    K, T = 6, 510.0
    _, Lout = O.fourier_llf(I, 3, K, T, 30.0, 2.0, return_output_pyramid=True)
    G, Ct, St = O.fourier_llf_pyramids(I, 3, K, T)
    c = O.fourier_coefficients(K, T, 30.0, 2.0)
    ref = I - O.up(G[1], I.shape)
    for k in range(K):
        w = c["omega"][k]
        ref = ref + c["a"][k] * (np.sin(w * I) * O.up(Ct[k][1], I.shape)
                                 - np.cos(w * I) * O.up(St[k][1], I.shape))
    assert np.abs(Lout[0] - ref).max() <= 1e-10


def test_explicit_coefficients_mode():
    I = _rand((15, 15), 10)
    c = O.fourier_coefficients(5, 510.0, 25.0, 1.5)
    a = O.fourier_llf(I, 3, 5, 510.0, 25.0, 1.5)
    b = O.fourier_llf(I, 3, 5, 510.0, a=c["a"])
    assert np.abs(a - b).max() <= 1e-12


def test_order_partition_sums_to_full():
    """Linearity of Eq. 4: sum over a partition of k = 1..K of the partial
    outputs (no base, top = 0) plus I equals the full output."""
    I = _rand((19, 22), 12)
    args = (4, 10, 510.0, 20.0, 2.0)
    full = O.fourier_llf(I, *args)
    parts = [O.fourier_llf(I, *args, k_range=r, include_base=False)
             for r in [(1, 4), (4, 8), (8, 11)]]
    assert np.abs(sum(parts) + I - full).max() <= 1e-9


# ------------------------------------------------------------------ adaptive
def test_adaptive_constant_maps_equal_scalar():
    I = _rand((20, 16), 13)
    s = np.full(I.shape, 30.0)
    mm = np.full(I.shape, 2.5)
    a = O.fourier_llf(I, 4, 12, 510.0, 30.0, 2.5)
    b = O.fourier_llf(I, 4, 12, 510.0, sigma_map=s, m_map=mm)
    assert np.abs(a - b).max() <= 1e-10


def test_adaptive_equals_naive_adaptive_truncated():
    """Exact identity for Sec. III-B: per-pixel coefficients at
    level l, pixel q == naive LLF whose remap at (l, q) is r_K with
    sigma_l(q), m_l(q) (reading R7)."""
    I = _rand((11, 9), 14)
    rng = np.random.default_rng(15)
    s = rng.uniform(10.0, 60.0, I.shape)
    mm = rng.uniform(0.5, 4.0, I.shape)
    F = O.fourier_llf(I, 3, 6, 510.0, sigma_map=s, m_map=mm)
    N = O.naive_llf_adaptive(I, 3, s, mm, K=6, T=510.0)
    assert np.abs(F - N).max() <= 1e-10
