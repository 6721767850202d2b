"""Golden values for the image-quality metrics (imaging.psnr / imaging.ssim,
imaging.py:249-311), produced by importing the real reference read-only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_metrics.py

Writes ``tests/golden/metrics_vectors.npz``: seeded input pairs (small f64
planes of several shapes, value ranges and noise levels) and the reference's
PSNR and SSIM for each.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "metrics_vectors.npz")

# (height, width, data_range, noise sigma as a fraction of the range)
CASES = [(11, 11, 1.0, 0.1), (15, 18, 255.0, 0.08), (37, 53, 1.0, 0.02), (64, 48, 2.0, 0.3),
         (96, 128, 255.0, 0.05)]


def main() -> None:
    sys.path.insert(0, REF)
    from noise2fast import imaging  # noqa: E402

    g = {}
    for k, (h, w, rng_, sig) in enumerate(CASES):
        r = np.random.default_rng(1000 + k)
        a = r.uniform(0, rng_, (h, w))
        b = a + r.normal(0, sig * rng_, (h, w))
        g[f"a{k}"], g[f"b{k}"] = a, b
        g[f"psnr{k}"] = np.float64(imaging.psnr(a, b, rng_))
        g[f"ssim{k}"] = np.float64(imaging.ssim(a, b, rng_))
        g[f"range{k}"] = np.float64(rng_)
    g["ncases"] = np.int64(len(CASES))
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, {k: float(v) for k, v in g.items() if k.startswith(("psnr", "ssim"))})


if __name__ == "__main__":
    main()
