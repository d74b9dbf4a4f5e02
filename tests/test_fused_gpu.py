"""Design F (materialise-once: the level-l order sum fused into the build step
l -> l+1, then the collapse over the D planes) against
the fp64 oracle, through fllf_filter (the call bench.py times).

Bar: max |GPU - oracle| <= 2e-3 (north star).  The fused build writes the
same G / Z planes as design AB (same arithmetic, checked bit for bit), and
F agrees with AB (build + apply) to fp32 rounding.
"""
import numpy as np
import pytest
import torch

from oracle import fllf_oracle as O
from paper_2206_04681_b200 import synth

pytestmark = pytest.mark.gpu

TOL_OUT = 2e-3
TOL_AB = 5e-4   # F vs AB: two fp32 evaluations of the same sums in different orders


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_04681_b200 import fllf
    return fllf


def maxerr(a, b):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max())


def run_both(F, x, levels, K, T, sig, m, pad=0, **kw):
    """(F output, AB output, plan launches of F) for x: (B, H, W) float32."""
    B, H, W = x.shape
    if pad:
        buf = torch.zeros((B, H, W + pad), dtype=torch.float32, device="cuda")
        buf[:, :, :W] = torch.from_numpy(x).cuda()
        d_in = buf[:, :, :W]
    else:
        d_in = torch.from_numpy(x).cuda()
    o_f = torch.full((B, H, W), float("nan"), device="cuda")
    o_ab = torch.full((B, H, W), float("nan"), device="cuda")
    with F.Plan(H, W, levels, K, T, sig, m, batch=B, design=F.FLLF_DESIGN_F, **kw) as p:
        p.filter(d_in, o_f)
        launches = p.launches
        p.build(d_in)
        p.apply(o_ab)
        torch.cuda.synchronize()
    return o_f.cpu().numpy().astype(np.float64), o_ab.cpu().numpy().astype(np.float64), launches


CASES = [
    # shape, levels, K, T, sigma_r, m, pad, batch
    ((37, 23), 3, 5, 510.0, 30.0, -1.5, 0, 1),     # odd sizes, K odd (1 order per warp), unaligned pitch
    ((50, 71), 4, 8, 510.0, 20.0, 3.0, 0, 1),
    ((9, 13), 3, 3, 405.9, 30.0, 7.0, 0, 1),       # tiny: coarsest 3x4, a single strip per level
    ((121, 300), 6, 16, 510.0, 10.0, 4.0, 5, 1),   # ragged + padded pitch, K = 16
    ((259, 130), 7, 1, 510.0, 60.0, 2.0, 3, 1),    # K = 1
    ((203, 347), 5, 32, 510.0, 30.0, 2.0, 0, 1),   # K = 32: 16 warps per CTA
    ((70, 119), 4, 12, 510.0, 25.0, 3.0, 0, 3),    # batch of 3 frames
    ((129, 257), 5, 10, 405.9, 20.0, 2.0, 0, 2),   # several column blocks, ragged tail
    ((64, 56), 3, 2, 510.0, 30.0, 3.0, 0, 1),      # one interior column block boundary
    ((300, 117), 4, 7, 510.0, 30.0, 3.0, 0, 1),    # tall: several strips per column block
]


@pytest.mark.parametrize("shape,levels,K,T,sig,m,pad,batch", CASES)
def test_fused_vs_oracle_and_ab(F, shape, levels, K, T, sig, m, pad, batch):
    x = np.stack([synth.uniform_image(*shape, seed=900 + 7 * K + i) for i in range(batch)]).astype(np.float32)
    of, oab, launches = run_both(F, x, levels, K, T, sig, m, pad)
    # design F: build0, l_max-1 fused, l_max-2 collapse, apply0 (2 l_max - 1 launches);
    # every order count up to 16 takes it (larger ones only when their shared memory fits)
    if K <= 16:
        assert launches == 2 * (levels - 1) - 1, launches
    else:
        assert launches in (2 * (levels - 1) - 1, 2 * (levels - 1)), launches
    for b in range(batch):
        ref = O.fourier_llf(x[b].astype(np.float64), levels, K, T, sig, m)
        assert maxerr(of[b], ref) <= TOL_OUT, b
    assert maxerr(of, oab) <= TOL_AB


def test_fused_pyramids_identical(F):
    """The fused kernel's build part is k_build's arithmetic: G_l and Z_{l,k}
    after fllf_filter equal those of fllf_build_fourier_pyramids bit for bit."""
    H, W, levels, K = 141, 233, 5, 6
    img = synth.uniform_image(H, W, seed=612)
    d_in = torch.from_numpy(img).cuda()
    out = torch.empty_like(d_in)
    planes = {}
    with F.Plan(H, W, levels, K, 510.0, 30.0, 3.0, design=F.FLLF_DESIGN_F) as p:
        for tag in ("F", "AB"):
            if tag == "F":
                p.filter(d_in, out)
            else:
                p.build(d_in)
            for l in range(1, levels):
                h, w = p.level_dims(l)
                for ch in range(K + 1):
                    t = torch.empty((h, w if ch == 0 else 2 * w), device="cuda")
                    p.read_pyramid(0, l, ch, t)
                    planes.setdefault((l, ch), []).append(t.cpu().numpy())
        torch.cuda.synchronize()
    for key, (a, b) in planes.items():
        assert np.array_equal(a, b), key


def test_fused_then_reapply(F):
    """fllf_filter (design F) leaves the plan built: a COEFFS apply afterwards
    (switch only the coefficients) matches the oracle."""
    H, W, levels, K = 96, 150, 4, 6
    img = synth.uniform_image(H, W, seed=613)
    a2 = np.linspace(2.0, -1.0, K)
    r1 = O.fourier_llf(img.astype(np.float64), levels, K, 510.0, 30.0, 2.0)
    r2 = O.fourier_llf(img.astype(np.float64), levels, K, 510.0, a=a2)
    d_in = torch.from_numpy(img).cuda()
    o = torch.empty_like(d_in)
    with F.Plan(H, W, levels, K, 510.0, 30.0, 2.0, design=F.FLLF_DESIGN_F) as p:
        p.filter(d_in, o)
        torch.cuda.synchronize()
        assert maxerr(o.cpu().numpy(), r1) <= TOL_OUT
        p.apply(o, mode=F.FLLF_COEFFS, a_k=a2)
        torch.cuda.synchronize()
        assert maxerr(o.cpu().numpy(), r2) <= TOL_OUT


@pytest.mark.parametrize("kb,ke,base", [(1, 4, False), (4, 8, False), (8, 11, True), (2, 3, False)])
def test_fused_order_range(F, kb, ke, base):
    """Order-sharded plans (config 3 layout) run design F too: the partial
    output of [kb, ke) with / without the base matches the oracle's."""
    img = synth.uniform_image(77, 190, seed=614)
    K, lev = 10, 5
    ref = O.fourier_llf(img.astype(np.float64), lev, K, 510.0, 20.0, 2.0, k_range=(kb, ke), include_base=base)
    of, oab, _ = run_both(F, img[None], lev, K, 510.0, 20.0, 2.0, k_begin=kb, k_end=ke, include_base=base)
    assert maxerr(of[0], ref) <= TOL_OUT
    assert maxerr(of, oab) <= TOL_AB


def test_fused_constant_and_identity(F):
    C = np.full((45, 62), 93.5, np.float32)
    of, _, _ = run_both(F, C[None], 4, 8, 510.0, 30.0, 3.0)
    assert maxerr(of[0], C) <= 1e-4
    img = synth.uniform_image(45, 62, seed=3)
    of, _, _ = run_both(F, img[None], 4, 8, 510.0, 30.0, 0.0)
    assert maxerr(of[0], img) <= 1e-4


def test_band_plans_reject_whole_pass_calls(F):
    """Row-band plans only run through the per-level calls (the halo rows of
    levels >= 1 are exchanged between them); the whole-pass calls refuse."""
    H, W, levels = 64, 40, 3
    img = torch.zeros((H, W), device="cuda")
    out = torch.zeros((32, W), device="cuda")
    with F.Plan(H, W, levels, 4, 510.0, 30.0, 2.0, row_begin=0, row_end=32) as p:
        for call in (lambda: p.filter(img, out), lambda: p.build(img), lambda: p.apply(out)):
            with pytest.raises(F.FllfError) as e:
                call()
            assert e.value.status == F.FLLF_ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("n", [1, 2, 3])
def test_mixed_fused_and_ab_levels(F, n):
    """Design F on levels 1..n and AB above (what FLLF_DESIGN_AUTO picks when
    only the fine levels are large): the sequence build0, fused 1..n, build /
    apply n+1.., collapse n..1, apply0 matches the oracle and pure AB."""
    H, W, levels, K = 150, 201, 6, 8
    img = synth.uniform_image(H, W, seed=615)
    ref = O.fourier_llf(img.astype(np.float64), levels, K, 510.0, 30.0, 3.0)
    d_in = torch.from_numpy(img).cuda()
    o_f = torch.full_like(d_in, float("nan"))
    o_ab = torch.full_like(d_in, float("nan"))
    with F.Plan(H, W, levels, K, 510.0, 30.0, 3.0) as p:
        F.fllf_plan_set_fused_levels(p.handle, n)
        p.filter(d_in, o_f)
        lmax = levels - 1
        assert p.launches == 1 + n + 2 * (lmax - 1 - n) + (min(n + 1, lmax - 1) - 1) + 1, p.launches
        p.set_design(F.FLLF_DESIGN_AB)
        p.filter(d_in, o_ab)
        assert p.launches == 2 * lmax
        torch.cuda.synchronize()
    assert maxerr(o_f.cpu().numpy(), ref) <= TOL_OUT
    assert maxerr(o_f.cpu().numpy(), o_ab.cpu().numpy()) <= TOL_AB


def test_design_api_errors(F):
    with F.Plan(64, 64, 3, 4) as p:
        with pytest.raises(F.FllfError):
            F.fllf_plan_set_design(p.handle, 7)
        with pytest.raises(F.FllfError):
            F.fllf_plan_set_fused_levels(p.handle, -1)
        d = F.fllf_plan_get_desc(p.handle)
        assert (d["H"], d["W"], d["levels"], d["K"], d["batch"], d["k_begin"], d["k_end"]) == (64, 64, 3, 4, 1, 1, 5)
        with pytest.raises(ValueError):   # shape checks of the binding
            p.filter(torch.zeros((64, 60), device="cuda"), torch.zeros((64, 64), device="cuda"))
