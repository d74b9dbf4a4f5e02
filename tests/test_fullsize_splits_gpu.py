"""Full-size parity of every split execution against the fp64 oracle
("complete full-size parity"):

* config 5: ALL 64 frames of the 64-frame batch, in the launch configuration
  bench.py times (one batched plan, fllf_filter, design chosen by AUTO);
* config 4: ALL 10 (sigma_r, m) map pairs, pyramids built once and reapplied
  (Sec. III-B: the pyramids do not depend on the maps);
* config 3: the order partition of 2, 4 and 8 ranks (order_partition /
  channel_runs, one plan per rank's run, emulated on one GPU), combined by a
  sum of the partial outputs (the NCCL reduce) and by the fused combine
  (fllf_apply_accumulate into one zeroed output), at 2160x3840x3;
* row bands: 2 and 4 bands of a 2160x3840 frame (band plans, per-level calls
  with the halo rows exchanged) vs the oracle.

Bar: max |GPU - oracle| <= 2e-3 per frame / channel / map (north star).  The
oracle calls run in parallel host processes and are cached
(tests/fllf_testutil.py).
"""
import numpy as np
import pytest
import torch

from fllf_testutil import oracle_many
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


def test_config5_all_frames(F):
    c = synth.CONFIGS[5]
    frames = synth.config5_frames(64)
    d_in = torch.from_numpy(frames).cuda()
    out = torch.full_like(d_in, float("nan"))
    with F.Plan(c["H"], c["W"], c["levels"], c["K"], c["T"], c["sigma_r"], c["m"], batch=64) as p:
        p.filter(d_in, out)
        torch.cuda.synchronize()
    got = out.cpu().numpy()
    refs = oracle_many("fourier_llf", [dict(img=frames[f], levels=c["levels"], K=c["K"], T=c["T"],
                                            sigma_r=c["sigma_r"], m=c["m"]) for f in range(64)])
    errs = [maxerr(got[f], refs[f]) for f in range(64)]
    assert max(errs) <= TOL_OUT, (int(np.argmax(errs)), max(errs))


def test_config4_all_maps(F):
    c = synth.CONFIGS[4]
    img = synth.config2_image(seed=4000, H=c["H"], W=c["W"])
    maps = [synth.config4_maps(j) for j in range(c["maps"])]
    refs = oracle_many("fourier_llf", [dict(img=img, levels=c["levels"], K=c["K"], T=c["T"],
                                            sigma_map=s.astype(np.float64), m_map=m.astype(np.float64))
                                       for s, m in maps])
    d_in = torch.from_numpy(img).cuda()
    out = torch.empty_like(d_in)
    with F.Plan(c["H"], c["W"], c["levels"], c["K"], c["T"], 30.0, 1.0) as p:
        p.build(d_in)                      # once
        for j, (s, m) in enumerate(maps):
            out.fill_(float("nan"))
            p.apply(out, mode=F.FLLF_MAPS, sigma_map=torch.from_numpy(s).cuda(), m_map=torch.from_numpy(m).cuda())
            torch.cuda.synchronize()
            assert maxerr(out.cpu().numpy(), refs[j]) <= TOL_OUT, j


@pytest.fixture(scope="module")
def config3_case():
    c = synth.CONFIGS[3]
    rgb = synth.config3_rgb()
    refs = oracle_many("fourier_llf", [dict(img=rgb[ch], levels=c["levels"], K=c["K"], T=c["T"],
                                            sigma_r=c["sigma_r"], m=c["m"]) for ch in range(3)])
    return c, rgb, refs


@pytest.mark.parametrize("P", [2, 4, 8])
def test_config3_order_partition(F, config3_case, P):
    """Every rank's runs of (channel, order) units (channel_runs: one batched
    plan per run) with its own order range and base flag; the sum over ranks
    is the reduce of the multi-GPU path.  The same plans then add their
    partials straight into one zeroed output (the fused combine's kernel)."""
    from paper_2206_04681_b200 import dist as D
    c, rgb, refs = config3_case
    C, H, W = rgb.shape
    img = torch.from_numpy(rgb).cuda()
    total = torch.zeros((C, H, W), dtype=torch.float32, device="cuda")
    acc = torch.zeros((C, H, W), dtype=torch.float32, device="cuda")
    part = torch.empty((C, H, W), dtype=torch.float32, device="cuda")
    for segs in D.order_partition(C, c["K"], P):
        for r in D.channel_runs(segs):
            with F.Plan(H, W, c["levels"], c["K"], c["T"], c["sigma_r"], c["m"], batch=r.nch, k_begin=r.k_begin,
                        k_end=r.k_end, include_base=r.include_base) as p:
                src = img[r.channel:r.channel + r.nch]
                dst = part[r.channel:r.channel + r.nch]
                p.filter(src, dst)
                total[r.channel:r.channel + r.nch] += dst
                F.fllf_apply_accumulate(p.handle, acc[r.channel:r.channel + r.nch])
        torch.cuda.synchronize()
    got, got_acc = total.cpu().numpy(), acc.cpu().numpy()
    for ch in range(C):
        assert maxerr(got[ch], refs[ch]) <= TOL_OUT, ("reduce", P, ch)
        assert maxerr(got_acc[ch], refs[ch]) <= TOL_OUT, ("accumulate", P, ch)


@pytest.mark.parametrize("P", [2, 4])
def test_bands_4k_vs_oracle(F, config3_case, P):
    from paper_2206_04681_b200 import dist as D
    c, rgb, refs = config3_case
    H, W = rgb.shape[1:]
    img = torch.from_numpy(np.ascontiguousarray(rgb[0])).cuda()
    out = torch.full((H, W), float("nan"), device="cuda")
    bands = [D.GpuBand(H, W, c["levels"], c["K"], c["T"], c["sigma_r"], c["m"], b)
             for b in D.band_partition(H, c["levels"], P)]
    try:
        D.band_filter_local(bands, img, out)
        torch.cuda.synchronize()
    finally:
        for b in bands:
            b.close()
    assert maxerr(out.cpu().numpy(), refs[0]) <= TOL_OUT
