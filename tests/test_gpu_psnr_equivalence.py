"""PSNR equivalence of full default fits against the STOCK reference
(north_star: "final denoised PSNR ... within 0.1 dB").

The fit is chaotic: the reference against ITSELF with
1e-7 relative init noise moves a single image's final PSNR by up to +-1 dB, so
the bar is a statement about the MEAN gap over many paired fits.  The CPU side
(hundreds of ~2-10 minute fits of the unmodified reference) was run once by
tools/psnr_equiv_cpu.py and is committed as tests/golden/psnr_reference_fits.json
(tests/golden/make_psnr_golden.py); here the engine fits the same seeded images
with the same TrainConfig and the paired gaps are tested:

  * the images are the same (noisy-image PSNR equal to 1e-9 dB);
  * every fit denoises (> +1 dB; the reference itself gains only +2.9 dB on
    the hardest 64^2 image) and stops by patience;
  * no single gap beyond 3.5 dB (the reference's own chaos partner stays
    within ~1.3 dB; the largest GPU gap measured is 2.1 dB);
  * per image size the mean gap does not contradict the bar: its 95 %
    confidence interval reaches into +-0.1 dB and the mean itself is within
    +-0.2 dB (the gap spread grows with the image size, sd 0.36 dB at 64^2 and
    0.65 dB at 128^2, so a single stratum's interval is wider than the bar
    below ~200 pairs);
  * the equivalence statement proper: the inverse-variance pooled mean over
    the sizes has its whole 95 % confidence interval inside +-0.1 dB.

GPU fits are bitwise reproducible, so this test is deterministic for a given
build.
"""

import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "psnr_reference_fits.json")
BAR_DB = 0.1


def _psnr(a, b):
    return 10 * np.log10(1.0 / np.mean((np.asarray(a, np.float64) - b) ** 2))


def _fit_gaps(key, fits):
    from paper_2108_10209_b200 import TrainConfig, synthetic, train_single_channel

    family, size = key.split(":")
    size = int(size)
    gaps = []
    for seed_s, ref in fits.items():
        seed = int(seed_s)
        if family == "config1":
            noisy, clean = synthetic.config_image(1, seed)
            noisy = noisy.astype(np.float64)
        else:
            clean = synthetic.blob_rect_image(size, size, 100 + seed)
            noisy = synthetic.gaussian_noisy(clean, 25 / 255, 200 + seed).astype(np.float64)
        p_in = _psnr(noisy, clean)
        assert abs(p_in - ref["psnr_noisy"]) < 1e-9, (key, seed, p_in, ref["psnr_noisy"])
        r = train_single_channel(noisy, TrainConfig(seed=seed))
        p = _psnr(r.denoised, clean)
        assert r.stop_reason == "patience" and p > p_in + 1.0, (key, seed, p, r.stop_reason)
        assert abs(p - ref["psnr"]) <= 3.5, (key, seed, p, ref["psnr"], r.epochs_run, ref["epochs"])
        gaps.append(p - ref["psnr"])
    return np.asarray(gaps)


def test_mean_psnr_gap_to_stock_reference_within_bar():
    fits = json.load(open(GOLDEN))["fits"]
    strata = []
    for key, rows in fits.items():
        if len(rows) < 30:  # too few pairs for a mean (e.g. the config-1 image): checked per image only
            _fit_gaps(key, rows)
            continue
        g = _fit_gaps(key, rows)
        mean, se = float(g.mean()), float(g.std(ddof=1) / math.sqrt(len(g)))
        print(f"{key}: n={len(g)} mean gap {mean:+.4f} dB, se {se:.4f}, sd {g.std(ddof=1):.3f}, "
              f"max |gap| {np.abs(g).max():.2f}")
        half = 1.96 * se
        assert mean - half <= BAR_DB and mean + half >= -BAR_DB and abs(mean) <= 2 * BAR_DB, (key, mean, se)
        strata.append((mean, se))
    assert strata
    w = np.array([1.0 / (se * se) for _, se in strata])
    m = np.array([mean for mean, _ in strata])
    pooled, pooled_se = float((w * m).sum() / w.sum()), float(1.0 / math.sqrt(w.sum()))
    lo, hi = pooled - 1.96 * pooled_se, pooled + 1.96 * pooled_se
    print(f"pooled (inverse-variance): {pooled:+.4f} dB, 95 % CI [{lo:+.4f}, {hi:+.4f}]")
    assert -BAR_DB <= lo and hi <= BAR_DB, (pooled, lo, hi)
