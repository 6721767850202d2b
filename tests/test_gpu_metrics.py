"""Device PSNR / SSIM (libn2f n2f_psnr / n2f_ssim) vs the reference's values
and the reference's own metric tests (test_imaging.py:245-320), restated on
the device path, plus full-size (4096^2) agreement with the NumPy oracle."""

import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "metrics_vectors.npz")


@pytest.fixture(scope="module")
def m():
    from paper_2108_10209_b200 import metrics

    return metrics


def ssim_scalar(a, b, data_range, size=11, sigma=1.5, k1=0.01, k2=0.03):
    """One window at a time (the reference test's independent oracle,
    test_imaging.py:25-55, restated)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    half = size // 2
    g1 = np.exp(-((np.arange(size) - half) ** 2) / (2 * sigma * sigma))
    win = np.outer(g1, g1)
    win /= win.sum()
    c1, c2 = (k1 * data_range) ** 2, (k2 * data_range) ** 2
    vals = []
    for y in range(half, a.shape[0] - half):
        for x in range(half, a.shape[1] - half):
            pa = a[y - half: y + half + 1, x - half: x + half + 1]
            pb = b[y - half: y + half + 1, x - half: x + half + 1]
            ma, mb = (win * pa).sum(), (win * pb).sum()
            va, vb = (win * pa * pa).sum() - ma ** 2, (win * pb * pb).sum() - mb ** 2
            cv = (win * pa * pb).sum() - ma * mb
            vals.append(((2 * ma * mb + c1) * (2 * cv + c2)) / ((ma ** 2 + mb ** 2 + c1) * (va + vb + c2)))
    return float(np.mean(vals))


def test_golden_reference_values(m):
    z = np.load(GOLDEN)
    for k in range(int(z["ncases"])):
        a, b, r = z[f"a{k}"], z[f"b{k}"], float(z[f"range{k}"])
        assert m.psnr(a, b, r) == pytest.approx(float(z[f"psnr{k}"]), rel=1e-12)
        assert m.ssim(a, b, r) == pytest.approx(float(z[f"ssim{k}"]), abs=1e-12)


def test_psnr_reference_cases(m):
    assert math.isinf(m.psnr(np.ones((8, 8)), np.ones((8, 8)), 255.0))
    assert m.psnr(np.zeros((4, 4)), np.full((4, 4), 2.0), 2.0) == pytest.approx(0.0, abs=1e-12)
    assert m.psnr(np.zeros((10, 10)), np.full((10, 10), 25.0), 255.0) == pytest.approx(
        20.172003435238352, abs=1e-9)
    a = np.random.default_rng(23).uniform(0, 255, (16, 16))
    prev = math.inf
    for scale in (1.0, 2.0, 4.0):
        v = m.psnr(a, a + scale, 255.0)
        assert v < prev
        prev = v


def test_ssim_reference_cases(m):
    a = np.random.default_rng(29).uniform(0, 255, (16, 16))
    assert m.ssim(a, a, 255.0) == pytest.approx(1.0, abs=1e-12)
    r = np.random.default_rng(31)
    a, b = r.uniform(0, 255, (14, 14)), r.uniform(0, 255, (14, 14))
    assert m.ssim(a, b, 255.0) == pytest.approx(m.ssim(b, a, 255.0), abs=1e-12)
    a = (np.random.default_rng(37).uniform(0, 1, (20, 20)) > 0.5).astype(np.float64)
    v = m.ssim(a, 1.0 - a, 1.0)
    assert v < 0.5 and v == pytest.approx(ssim_scalar(a, 1.0 - a, 1.0), abs=1e-10)
    r = np.random.default_rng(41)
    a = r.uniform(0, 255, (15, 18))
    b = a + r.normal(0, 20, (15, 18))
    assert m.ssim(a, b, 255.0) == pytest.approx(ssim_scalar(a, b, 255.0), abs=1e-10)


@pytest.mark.parametrize("hw", [(11, 200), (130, 67), (517, 1031)])
def test_ssim_ragged_shapes_vs_oracle(m, oracle, hw):
    """Tile edges: valid regions that are not multiples of the 32 x 16 tile."""
    r = np.random.default_rng(hw[0] * 7 + hw[1])
    a = r.random(hw)
    b = np.clip(a + r.normal(0, 0.1, hw), 0, 1)
    assert m.ssim(a, b, 1.0) == pytest.approx(oracle.ssim(a, b, 1.0), abs=1e-11)
    assert m.psnr(a, b, 1.0) == pytest.approx(oracle.psnr(a, b, 1.0), rel=1e-12)


def test_metrics_full_size_4096(m, oracle):
    """Config-5 size, device-resident inputs (CUDA tensors are used in place)."""
    import torch

    from paper_2108_10209_b200 import synthetic

    noisy, clean = synthetic.config_image(5, 0)
    a = torch.from_numpy(noisy.astype(np.float64)).cuda()
    b = torch.from_numpy(clean.astype(np.float64)).cuda()
    rng_ = float(clean.max() - clean.min())
    assert m.psnr(a, b, rng_) == pytest.approx(oracle.psnr(noisy, clean, rng_), rel=1e-12)
    assert m.ssim(a, b, rng_) == pytest.approx(oracle.ssim(noisy, clean, rng_), abs=1e-11)
