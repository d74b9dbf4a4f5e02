"""fllf_apply_maps: n MAPS applies with the map pyramids of all n (sigma_r, m)
pairs built in one launch per level (Sec. III-B: the pyramids do
not depend on the maps).  Output j must equal fllf_apply(MAPS) with pair j bit
for bit (same kernels, same arithmetic; only the map-pyramid launches are
shared), and the fp64 oracle within the north star's 2e-3.
"""
import numpy as np
import pytest
import torch

from oracle import fllf_oracle as O
from paper_2206_04681_b200 import synth

pytestmark = pytest.mark.gpu

TOL_OUT = 2e-3


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_04681_b200 import fllf
    return fllf


def maxerr(a, b):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max())


def random_maps(n, H, W, seed):
    rng = np.random.default_rng(seed)
    s = rng.uniform(10.0, 60.0, (n, H, W)).astype(np.float32)
    m = rng.uniform(0.5, 4.0, (n, H, W)).astype(np.float32)
    return s, m


def per_map_and_batched(F, img, levels, K, T, s, m, batch=1):
    n, H, W = s.shape
    d_img = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    ds, dm = torch.from_numpy(s).cuda(), torch.from_numpy(m).cuda()
    shape = (n, batch, H, W) if batch > 1 else (n, H, W)
    single = torch.full(shape, float("nan"), device="cuda")
    batched = torch.full(shape, float("nan"), device="cuda")
    with F.Plan(H, W, levels, K, T, 30.0, 1.0, batch=batch) as p:
        p.build(d_img)
        for j in range(n):
            p.apply(single[j], mode=F.FLLF_MAPS, sigma_map=ds[j], m_map=dm[j])
        p.apply_maps(batched, ds, dm)
        # a single-pair apply after the batched call still works (slot 0)
        again = torch.full_like(single[0], float("nan"))
        p.apply(again, mode=F.FLLF_MAPS, sigma_map=ds[0], m_map=dm[0])
        torch.cuda.synchronize()
    return single.cpu().numpy(), batched.cpu().numpy(), again.cpu().numpy()


@pytest.mark.parametrize("shape,levels,K,n", [((90, 132), 5, 12, 3), ((77, 64), 4, 7, 2), ((41, 36), 3, 16, 4)])
def test_apply_maps_equals_per_map(F, shape, levels, K, n):
    H, W = shape
    img = synth.uniform_image(H, W, seed=H + W)
    s, m = random_maps(n, H, W, seed=n)
    single, batched, again = per_map_and_batched(F, img, levels, K, 510.0, s, m)
    assert np.array_equal(single, batched)
    assert np.array_equal(again, single[0])
    ref = O.fourier_llf(img.astype(np.float64), levels, K, 510.0, sigma_map=s[-1].astype(np.float64),
                        m_map=m[-1].astype(np.float64))
    assert maxerr(batched[-1], ref) <= TOL_OUT


def test_apply_maps_batch_frames(F):
    """A plan of 2 frames: every pair's maps apply to both frames."""
    H, W = 64, 96
    img = np.stack([synth.uniform_image(H, W, seed=7), synth.uniform_image(H, W, seed=8)])
    s, m = random_maps(2, H, W, seed=9)
    single, batched, _ = per_map_and_batched(F, img, 4, 8, 510.0, s, m, batch=2)
    assert np.array_equal(single, batched)


def test_apply_maps_config4_full(F):
    """BASELINE configs[3] size (2160x3840, 7 levels, K = 12), three of its map pairs."""
    c = synth.CONFIGS[4]
    img = synth.config2_image(seed=4000, H=c["H"], W=c["W"])
    pairs = [synth.config4_maps(j, H=c["H"], W=c["W"]) for j in (0, 4, 9)]
    s = np.stack([p[0] for p in pairs])
    m = np.stack([p[1] for p in pairs])
    single, batched, _ = per_map_and_batched(F, img, c["levels"], c["K"], c["T"], s, m)
    assert np.array_equal(single, batched)


def test_apply_maps_errors(F):
    H, W = 40, 48
    s = torch.rand(2, H, W, device="cuda") * 50 + 10
    m = torch.rand(2, H, W, device="cuda") + 1
    outs = torch.empty(2, H, W, device="cuda")
    with F.Plan(H, W, 3, 4, 510.0, 30.0, 1.0) as p:
        with pytest.raises(F.FllfError):
            p.apply_maps(outs, s, m)            # before a build
        p.build(torch.rand(H, W, device="cuda") * 255)
        with pytest.raises(ValueError):
            p.apply_maps(outs[:1], s, m)        # one output per pair
        p.apply_maps(outs, s, m)
        torch.cuda.synchronize()
        assert torch.isfinite(outs).all()
