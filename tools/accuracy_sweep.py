"""NEXT-2: accuracy of Fourier LLF against the naive-LLF ground truth as a
function of the number of pyramids (2K+1), for 2, 3 and 4 layers -- the
synthetic counterpart of the paper's Fig. 4(a) (the
paper's ten 512x512 test photographs are not available, so seeded 512x512
config-2-style images stand in for them).  sigma_r = 30; m is not
stated for Fig. 4 -- m = 2 here; T = 405.9 as in the paper
 and T*(K) from Eq. 12 (fllf_optimal_period).  Everything runs on the
GPU through the C ABI (fllf_filter and fllf_naive_llf).

    python tools/accuracy_sweep.py [--n-images 3] [--out profiles/r01_accuracy_sweep]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2206_04681_b200 import fllf as F  # noqa: E402
from paper_2206_04681_b200 import synth  # noqa: E402

SIGMA, M, N = 30.0, 2.0, 512
KS = [1, 2, 3, 4, 5, 6, 8, 10, 12, 16]


def psnr(a, b):
    mse = float(np.mean((a - b) ** 2))
    return float("inf") if mse == 0 else 10.0 * math.log10(255.0 ** 2 / mse)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-images", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_accuracy_sweep"))
    a = ap.parse_args()
    imgs = [torch.from_numpy(synth.config2_image(seed=7000 + i, H=N, W=N)).cuda() for i in range(a.n_images)]
    out = torch.empty_like(imgs[0])
    rows = []
    for levels in (2, 3, 4):
        truth = []
        with F.Plan(N, N, levels, 1, 510.0, SIGMA, M) as p:
            for im in imgs:
                F.fllf_naive_llf(p.handle, im, out, F.REMAP_EXACT)
                torch.cuda.synchronize()
                truth.append(out.cpu().numpy().astype(np.float64))
        for K in KS:
            for tname in ("405.9", "eq12"):
                T = 405.9 if tname == "405.9" else F.fllf_optimal_period(K, SIGMA, 256.0)
                vals = []
                with F.Plan(N, N, levels, K, T, SIGMA, M) as p:
                    for im, gt in zip(imgs, truth):
                        p.filter(im, out)
                        torch.cuda.synchronize()
                        vals.append(psnr(out.cpu().numpy().astype(np.float64), gt))
                rows.append({"layers": levels, "K": K, "pyramids": 2 * K + 1, "T": round(T, 2), "T_rule": tname,
                             "psnr_mean": round(float(np.mean(vals)), 2), "psnr_min": round(float(np.min(vals)), 2)})
                print(rows[-1], flush=True)
    t10 = F.fllf_optimal_period(10, SIGMA, 256.0)
    md = ["# NEXT-2: Fourier LLF accuracy vs number of pyramids (synthetic stand-in for Fig. 4(a))", "",
          f"{a.n_images} seeded {N}x{N} config-2-style images (the paper's test photographs are not available), "
          f"sigma_r = {SIGMA}, m = {M}; ground truth = naive LLF with the exact Gaussian remap "
          "(GPU `fllf_naive_llf`, parity-tested against the fp64 oracle); PSNR on the 0-255 scale, mean (min) "
          "over the images.", "",
          f"Eq. 12 optimal period for K = 10, sigma_r = 30, R = 256: T* = {t10:.2f} (paper: 405.9, P:296).", "",
          "| layers | K | pyramids (2K+1) | PSNR dB, T = 405.9 | PSNR dB, T = T*(K) (Eq. 12) | T*(K) |",
          "|---|---|---|---|---|---|"]
    for levels in (2, 3, 4):
        for K in KS:
            r1 = next(r for r in rows if r["layers"] == levels and r["K"] == K and r["T_rule"] == "405.9")
            r2 = next(r for r in rows if r["layers"] == levels and r["K"] == K and r["T_rule"] == "eq12")
            md.append(f"| {levels} | {K} | {2 * K + 1} | {r1['psnr_mean']:.2f} ({r1['psnr_min']:.2f}) | "
                      f"{r2['psnr_mean']:.2f} ({r2['psnr_min']:.2f}) | {r2['T']:.1f} |")
    open(a.out + ".md", "w").write("\n".join(md) + "\n")
    json.dump(rows, open(a.out + ".json", "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
