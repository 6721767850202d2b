"""`denoise_image` (trainer.py:216-250) on the engine: a 3-channel x 2-slice
image fans out into 6 independent fits with seeds derive_seed(seed, ch, sl)
(trainer.py:240), each checked against the CPU oracle's fit of the same plane
with the same derived seed (bounded fits: the first epoch inside the step
parity window, the short-fit bars of test_gpu_engine.py), and bitwise against
a solo train_single_channel call with that seed (the reference's own
test_stack_five_runs_order_preserved, test_trainer.py:342-354, restated)."""

import dataclasses

import numpy as np
import pytest

from n2f_testutil import norm_rel

pytestmark = pytest.mark.gpu


def test_denoise_image_fanout_matches_oracle(oracle):
    from paper_2108_10209_b200 import ImageData, TrainConfig, denoise_image, synthetic, train_single_channel
    from paper_2108_10209_b200 import trainer as T

    n_sl, h, w, n_ch = 2, 40, 36, 3
    samples = np.empty((n_sl, h, w, n_ch), np.float32)
    for sl in range(n_sl):
        for ch in range(n_ch):
            clean = synthetic.blob_rect_image(h, w, 50 + 10 * sl + ch)
            samples[sl, :, :, ch] = 255.0 * synthetic.gaussian_noisy(clean, 25 / 255, 70 + 10 * sl + ch)
    img = ImageData(samples, "uint8", 255.0)
    cfg = TrainConfig(seed=123, max_epochs=3, patience_epochs=50, avg_window=2)
    out, runs = denoise_image(img, cfg)
    assert out.samples.shape == samples.shape and out.samples.dtype == np.float32
    assert len(runs) == n_sl * n_ch
    k = 0
    for sl in range(n_sl):
        for ch in range(n_ch):
            seed = T.derive_seed(cfg.seed, ch, sl)
            assert seed == oracle.child_seed(cfg.seed, ch, sl)  # rng.py:31-39
            plane = samples[sl, :, :, ch].astype(np.float64)
            ref = oracle.fit_denoise(plane, seed=seed, patience=50, window=2, max_epochs=3)
            r = runs[k]
            k += 1
            assert r.epochs_run == ref.epochs_run == 3
            assert abs(r.val_history[0] - ref.val_history[0]) <= 5e-3 * ref.val_history[0]
            assert norm_rel(out.samples[sl, :, :, ch], ref.denoised) < 2e-2
            solo = train_single_channel(samples[sl, :, :, ch], dataclasses.replace(cfg, seed=seed))
            assert np.array_equal(out.samples[sl, :, :, ch], solo.denoised.astype(np.float32))
    T.release_engines()

