"""Fourier local Laplacian filtering -- the fp64 CPU ORACLE.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call or
execute this module: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` use it.  It shares
no code, header, table or constant generator with the CUDA path
(``paper_2206_04681_b200/csrc``), and imports nothing from it.

What it is: a plain, slow, obviously-correct numpy float64 implementation of
the paper "Gaussian Fourier Pyramid for Local Laplacian Filter"
(Sumiya, Otsuka, Maeda, Fukushima; arXiv 2206.04681), following the paper's
equations step by step in the paper's notation.  Citations "P:n" are
``/root/reference/PAPER.md`` line numbers (section / equation given with each).
No blocking, fusion or reordering is applied beyond what the equations state;
library primitives used as steps: ``numpy.take`` (gather), elementwise
arithmetic, ``numpy.sin/cos/exp``, ``math.erfc``.

Readings of places where the paper is silent, ambiguous or garbled (each is
listed in DESIGN.md, "Readings of the paper"):

R1  Remap sign.  Eq. 5 as printed, r = i - (i-g) f(i-g), smooths for
    m>0, contradicting P:184 ("m>0 enhances").  Eq. 7 drops the minus
    sign of the Gaussian derivative; the two slips cancel and Eq. 11
    and Eq. 14 are the ENHANCING remap
        r(i,g) = i + m (i-g) exp(-(i-g)^2 / (2 sigma_r^2)).
    This is the sign BASELINE.json's north star fixes.  ``remap_exact`` uses it.
R2  Borders: the paper states none.  Reflect-101 (index -j -> j,
    n-1+j -> n-1-j, bounced until in range) for both down- and up-sampling.
R3  Odd sizes: ceil-halving (P:107-108 says "halves"), the up-sampling
    targets the recorded finer size.
R4  "Layers" == number of pyramid levels including the residual
    (levels = 2 -> one detail level).  l_max = levels - 1.
R5  Up-sampling kernel = 2x the 5-tap binomial per axis after zero insertion
    ("Usually, the kernel is identical to G_sigma"; the factor 2
    per axis keeps a constant image fixed).
R6  Coefficients at level l use g = G_l[I]_p for BOTH the same-level and the
    up-sampled next-level terms, exactly as Eq. 14 is printed.
R7  Per-pixel parameter maps at level l are read from the
    Gaussian pyramid of each map (the paper does not say how a full-resolution
    map is looked up at a coarse level).
R8  No clamping or quantisation anywhere; outputs are raw floats.
R9  The 5-tap kernel is the binomial [1,4,6,4,1]/16 ("binomial
    distribution ... with five taps", sigma ~ 1).
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "BINOMIAL5", "reflect101", "down", "up", "gaussian_pyramid",
    "laplacian_pyramid", "collapse", "level_shapes", "fourier_coefficients",
    "remap_exact", "remap_fourier", "fourier_llf", "fourier_llf_pyramids",
    "naive_llf", "naive_llf_adaptive", "period_error", "optimal_period",
]

# P:109-110 (Sec. II-A): "the Gaussian convolution is based on the binomial
# distribution for integer operations with five taps ... sigma = 1" (R9).
BINOMIAL5 = np.array([1.0, 4.0, 6.0, 4.0, 1.0]) / 16.0
_TAPS = (-2, -1, 0, 1, 2)


def reflect101(idx, n: int):
    """Reflect-101 border (R2): -j -> j, (n-1)+j -> (n-1)-j, bounced until the
    index is inside [0, n-1].  Bouncing forever is folding with period 2(n-1)."""
    idx = np.asarray(idx)
    if n == 1:
        return np.zeros_like(idx)
    period = 2 * (n - 1)
    r = np.mod(idx, period)
    return np.where(r < n, r, period - r)


def _down_axis(x: np.ndarray, axis: int) -> np.ndarray:
    """out(o) = sum_j w_j x(refl(2o + j)), o = 0 .. ceil(n/2)-1  (Eq. 1 along one axis)."""
    n = x.shape[axis]
    o = np.arange((n + 1) // 2)
    out = 0.0
    for j, w in zip(_TAPS, BINOMIAL5):
        out = out + w * np.take(x, reflect101(2 * o + j, n), axis=axis)
    return out


def down(x: np.ndarray) -> np.ndarray:
    """(G_sigma * X)_down of Eq. 1: separable 5-tap binomial blur,
    reflect-101 borders, keep even rows and columns (ceil-halving, R3).
    1-D input is filtered along its only axis."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        return _down_axis(x, 0)
    return _down_axis(_down_axis(x, 1), 0)


def _up_axis(x: np.ndarray, n: int, axis: int) -> np.ndarray:
    """Zero-insert to length n (z(2c) = x(c), odd samples 0), then
    out(t) = sum_j 2 w_j z(refl(t + j)) with the reflection on the FINE grid."""
    c = x.shape[axis]
    if c != (n + 1) // 2:
        raise ValueError(f"up: coarse size {c} does not match fine size {n}")
    shape = list(x.shape)
    shape[axis] = n
    z = np.zeros(shape)
    sl = [slice(None)] * x.ndim
    sl[axis] = slice(0, n, 2)
    z[tuple(sl)] = x
    t = np.arange(n)
    out = 0.0
    for j, w in zip(_TAPS, BINOMIAL5):
        out = out + 2.0 * w * np.take(z, reflect101(t + j, n), axis=axis)
    return out


def up(x: np.ndarray, shape) -> np.ndarray:
    """The up-sampling operator of Eq. 2 to the recorded fine
    ``shape`` (R3, R5).  1-D input takes ``shape = (n,)`` or ``n``."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        return _up_axis(x, int(shape[0]) if np.ndim(shape) else int(shape), 0)
    return _up_axis(_up_axis(x, shape[1], 1), shape[0], 0)


def level_shapes(shape, levels: int):
    """Dimensions of levels 0..l_max under ceil-halving (R3)."""
    shapes = [tuple(shape)]
    for _ in range(levels - 1):
        h, w = shapes[-1]
        shapes.append(((h + 1) // 2, (w + 1) // 2))
    return shapes


def gaussian_pyramid(img: np.ndarray, levels: int):
    """G_0 = I, G_l = (G_sigma * G_{l-1})_down  (Eq. 1)."""
    G = [np.asarray(img, dtype=np.float64)]
    for _ in range(1, levels):
        G.append(down(G[-1]))
    return G


def laplacian_pyramid(img: np.ndarray, levels: int):
    """L_l = G_l - (G_{l+1})_up (Eq. 2); L_lmax = G_lmax."""
    G = gaussian_pyramid(img, levels)
    L = [G[l] - up(G[l + 1], G[l].shape) for l in range(levels - 1)]
    L.append(G[-1])
    return L


def collapse(L):
    """O = sum_l L_l with up-sample-and-add from the coarsest level (Eq. 4)."""
    O = np.asarray(L[-1], dtype=np.float64)
    for l in range(len(L) - 2, -1, -1):
        O = L[l] + up(O, L[l].shape)
    return O


def fourier_coefficients(K: int, T: float, sigma_r: float, m: float = 1.0):
    """Eq. 9-11:
        omega_k = 2 pi k / T,
        alpha_k = sigma_r sqrt(2 pi)/T * exp(-(omega_k sigma_r)^2 / 2),
        alpha~_k = 2 sigma_r^2 alpha_k omega_k,
    and a_k = m alpha~_k, so that (R1)
        r(i,g) ~= i + sum_{k=1..K} a_k sin(omega_k (i - g)).
    Returns arrays indexed k = 1..K (alpha_0 separately; it is unused, Eq. 10)."""
    k = np.arange(0, K + 1, dtype=np.float64)
    omega = 2.0 * math.pi * k / T
    alpha = sigma_r * math.sqrt(2.0 * math.pi) / T * np.exp(-0.5 * (omega * sigma_r) ** 2)
    alpha_t = 2.0 * sigma_r ** 2 * alpha * omega
    return {
        "omega": omega[1:], "alpha0": float(alpha[0]), "alpha": alpha[1:],
        "alpha_tilde": alpha_t[1:], "a": m * alpha_t[1:],
    }


def remap_exact(i, g, sigma_r: float, m: float):
    """Eq. 5-6 with the enhancing sign of R1:  r(i,g) = i + m (i-g) exp(-(i-g)^2/(2 sigma_r^2))."""
    d = np.asarray(i, dtype=np.float64) - g
    return i + m * d * np.exp(-(d * d) / (2.0 * sigma_r ** 2))


def remap_fourier(i, g, a, omega):
    """Eq. 11, written with the addition theorem undone:
    r_K(i,g) = i - sum_k a_k (sin(w_k g) cos(w_k i) - cos(w_k g) sin(w_k i))
             = i + sum_k a_k sin(w_k (i - g))."""
    i = np.asarray(i, dtype=np.float64)
    out = np.array(i, dtype=np.float64, copy=True)
    for ak, wk in zip(a, omega):
        out = out - ak * (np.sin(wk * g) * np.cos(wk * i) - np.cos(wk * g) * np.sin(wk * i))
    return out


def _level_coefficients(K, T, levels, shape, sigma_r, m, a, sigma_map, m_map):
    """Per-level coefficient arrays a_{l,k} (scalar, explicit, or per-pixel).
    Per-pixel (Sec. III-B; R7): sigma_l = G_l[sigma map],
    m_l = G_l[m map], a_{l,k}(q) = m_l(q) * 2 sigma_l(q)^2 omega_k *
    (sigma_l(q) sqrt(2 pi)/T) exp(-(omega_k sigma_l(q))^2/2)."""
    omega = 2.0 * math.pi * np.arange(1, K + 1) / T
    if sigma_map is not None or m_map is not None:
        if sigma_map is None or m_map is None:
            raise ValueError("per-pixel mode needs both sigma_r and m maps")
        S = gaussian_pyramid(sigma_map, levels)
        M = gaussian_pyramid(m_map, levels)
        per_level = []
        for l in range(levels):
            s = S[l]
            ak = []
            for wk in omega:
                alpha = s * math.sqrt(2.0 * math.pi) / T * np.exp(-0.5 * (wk * s) ** 2)
                ak.append(M[l] * 2.0 * s ** 2 * alpha * wk)
            per_level.append(ak)
        return omega, per_level
    if a is None:
        a = fourier_coefficients(K, T, sigma_r, m)["a"]
    a = np.asarray(a, dtype=np.float64)
    if a.shape != (K,):
        raise ValueError("explicit coefficients must hold exactly K values")
    return omega, [list(a) for _ in range(levels)]


def fourier_llf_pyramids(img, levels, K, T):
    """The 2K+1 pyramids of P:262: G_l[I], C~_{l,k} = G_l[cos(omega_k I)] and
    S~_{l,k} = G_l[sin(omega_k I)], k = 1..K, levels 0..l_max.
    Full-resolution cos/sin images are materialised (general form)."""
    I = np.asarray(img, dtype=np.float64)
    omega = 2.0 * math.pi * np.arange(1, K + 1) / T
    G = gaussian_pyramid(I, levels)
    Ct = [gaussian_pyramid(np.cos(wk * I), levels) for wk in omega]
    St = [gaussian_pyramid(np.sin(wk * I), levels) for wk in omega]
    return G, Ct, St


def fourier_llf(img, levels, K, T, sigma_r=None, m=None, a=None,
                sigma_map=None, m_map=None, k_range=None, include_base=True,
                return_output_pyramid=False):
    """Fourier LLF, Eq. 13-14 and Fig. 1, collapsed by Eq. 4.

    For every level 0 <= l <= l_max-1, with g = G_l[I] pointwise (R6):
      L_l[O] = G_l[I] - m sum_k alpha~_k (sin(w_k g) C~_{l,k} - cos(w_k g) S~_{l,k})
               - G_{l+1}[I]_up
               + m sum_k alpha~_k (sin(w_k g) C~_{l+1,k,up} - cos(w_k g) S~_{l+1,k,up})
    with m alpha~_k replaced by a_k (scalar, given, or per pixel, Sec. III-B).
    The same general form is used at l = 0 (C~_{0,k} = cos(w_k I)); the paper's
    reduced l = 0 case follows from it because the same-level term
    vanishes there (sin(w I)cos(w I) - cos(w I)sin(w I) = 0), which is checked
    by a pin, not assumed.  L_lmax[O] = G_lmax[I].

    ``k_range=(k0,k1)`` keeps only the Fourier terms k0 <= k < k1 (1-based);
    ``include_base=False`` drops G_l - G_{l+1,up} and the top level, so that
    sum over a partition of 1..K of the partial outputs + I equals the full
    output (linearity of Eq. 4; used by order-sharding).
    """
    I = np.asarray(img, dtype=np.float64)
    if levels < 2:
        raise ValueError("levels must be >= 2")
    lmax = levels - 1
    omega, coef = _level_coefficients(K, T, levels, I.shape, sigma_r, m, a,
                                      sigma_map, m_map)
    k0, k1 = (1, K + 1) if k_range is None else k_range
    G, Ct, St = fourier_llf_pyramids(I, levels, K, T)
    Lout = []
    for l in range(lmax):
        shape = G[l].shape
        g = G[l]
        if include_base:
            Ll = G[l] - up(G[l + 1], shape)
        else:
            Ll = np.zeros(shape)
        same = np.zeros(shape)
        upper = np.zeros(shape)
        for k in range(k0, k1):
            wk = omega[k - 1]
            ak = coef[l][k - 1]
            sin_g = np.sin(wk * g)
            cos_g = np.cos(wk * g)
            same = same + ak * (sin_g * Ct[k - 1][l] - cos_g * St[k - 1][l])
            upper = upper + ak * (sin_g * up(Ct[k - 1][l + 1], shape)
                                  - cos_g * up(St[k - 1][l + 1], shape))
        Lout.append(Ll - same + upper)
    Lout.append(G[lmax] if include_base else np.zeros(G[lmax].shape))
    O = collapse(Lout)
    return (O, Lout) if return_output_pyramid else O


def naive_llf(img, levels, remap):
    """Naive LLF, Sec. II-C steps 1-5.  For every level l < l_max
    and every pixel q of level l: g = G_l[I]_q, remap the WHOLE image
    I~ = r(I, g), build its pyramid and copy L_l[I~]_q (Eq. 13);
    L_lmax[O] = G_lmax[I]; collapse (Eq. 4).  ``remap(I, g, l, q)`` returns the
    remapped full-resolution image.  O(N^2) -- tiny images only."""
    I = np.asarray(img, dtype=np.float64)
    lmax = levels - 1
    G = gaussian_pyramid(I, levels)
    Lout = []
    for l in range(lmax):
        Ll = np.zeros(G[l].shape)
        for q in np.ndindex(*G[l].shape):
            Ir = remap(I, G[l][q], l, q)
            Gr = gaussian_pyramid(Ir, l + 2)
            Ll[q] = Gr[l][q] - up(Gr[l + 1], Gr[l].shape)[q]
        Lout.append(Ll)
    Lout.append(G[lmax])
    return collapse(Lout)


def naive_llf_adaptive(img, levels, sigma_map, m_map, K=None, T=None):
    """Pixel-by-pixel naive LLF (Sec. III-B): at level l and pixel q
    the remap uses sigma_l(q) = G_l[sigma map]_q and m_l(q) = G_l[m map]_q (R7);
    with K,T given the remap is the truncated series r_K, else the exact one."""
    S = gaussian_pyramid(sigma_map, levels)
    M = gaussian_pyramid(m_map, levels)

    def remap(I, g, l, q):
        s, mm = float(S[l][q]), float(M[l][q])
        if K is None:
            return remap_exact(I, g, s, mm)
        c = fourier_coefficients(K, T, s, mm)
        return remap_fourier(I, g, c["a"], c["omega"])

    return naive_llf(img, levels, remap)


def period_error(T: float, K: int, sigma: float, R: float) -> float:
    """Eq. 12: E_K(T) = erfc(pi sigma (2K+1)/T) + erfc((T-R)/sigma)."""
    return math.erfc(math.pi * sigma * (2 * K + 1) / T) + math.erfc((T - R) / sigma)


def optimal_period(K: int, sigma: float, R: float = 256.0, tol: float = 1e-6) -> float:
    """argmin_T E_K(T) (Eq. 12): dense grid over [R, R + 12 sigma], then
    golden-section refinement around the best grid point."""
    lo, hi = float(R), float(R) + 12.0 * sigma
    grid = np.linspace(lo, hi, 4001)
    vals = [period_error(t, K, sigma, R) for t in grid]
    i = int(np.argmin(vals))
    a, b = grid[max(i - 1, 0)], grid[min(i + 1, len(grid) - 1)]
    phi = (math.sqrt(5.0) - 1.0) / 2.0
    c, d = b - phi * (b - a), a + phi * (b - a)
    while b - a > tol:
        if period_error(c, K, sigma, R) < period_error(d, K, sigma, R):
            b, d = d, c
            c = b - phi * (b - a)
        else:
            a, c = c, d
            d = a + phi * (b - a)
    return 0.5 * (a + b)
