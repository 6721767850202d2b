"""Seeded synthetic inputs for BASELINE.json's configs.

These stand in for the paper's BSD68 / Set12 / FMD data (not available
offline): blob+rectangle scenes with additive Gaussian noise from the
reference's counter RNG stream (imaging.add_gaussian_noise,
imaging.py:171-182: N(0, sigma^2) from CounterRng(derive_seed(seed, "nois")),
unclipped), and a microscopy-like puncta+filament scene with Poisson shot
noise plus Gaussian read noise (config 3).  Rectangle extents, polyline
vertex counts and the Poisson/Gaussian seeds are fixed here.
"""

from __future__ import annotations

import numpy as np

from .trainer import derive_seed

_M64 = 0xFFFFFFFFFFFFFFFF


def _mix(words: np.ndarray) -> np.ndarray:
    z = np.asarray(words, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def counter_normal(seed: int, n: int, sigma: float = 1.0) -> np.ndarray:
    """Box-Muller normals on 53-bit counter uniforms (rng.py:66-78)."""
    half = (n + 1) // 2
    key = _mix(np.array([seed & _M64], dtype=np.uint64))[0]
    u = (_mix(np.arange(0, 2 * half, dtype=np.uint64) ^ key) >> np.uint64(11)).astype(np.float64)
    u *= float(2.0**-53)
    rad = np.sqrt(-2.0 * np.log(1.0 - u[:half]))
    ang = 2.0 * np.pi * u[half:]
    return np.concatenate([rad * np.cos(ang), rad * np.sin(ang)])[:n] * sigma


def blob_rect_image(h: int, w: int, seed: int, n_blobs: int = 20, n_rects: int = 5) -> np.ndarray:
    """Clean blob+rectangle scene in [0,1] (configs 1, 2, 4, 5)."""
    r = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    img = np.zeros((h, w))
    # large images (config 5) evaluate each blob inside a +-10 sigma window
    # only (exp(-50) ~ 2e-22: below float32 resolution of any pixel it touches)
    windowed = h * w > (1 << 22)
    for _ in range(n_blobs):
        cy, cx = r.uniform(0, h), r.uniform(0, w)
        amp, sg = r.uniform(0.2, 1.0), r.uniform(4, 30)
        if windowed:
            y0, y1 = max(0, int(cy - 10 * sg)), min(h, int(cy + 10 * sg) + 1)
            x0, x1 = max(0, int(cx - 10 * sg)), min(w, int(cx + 10 * sg) + 1)
            img[y0:y1, x0:x1] += amp * np.exp(
                -((yy[y0:y1, x0:x1] - cy) ** 2 + (xx[y0:y1, x0:x1] - cx) ** 2) / (2 * sg * sg))
            continue
        img += amp * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * sg * sg))
    for _ in range(n_rects):
        y0, x0 = int(r.integers(0, h - 8)), int(r.integers(0, w - 8))
        rh, rw = int(r.integers(8, max(9, h // 4))), int(r.integers(8, max(9, w // 4)))
        img[y0 : y0 + rh, x0 : x0 + rw] = r.uniform(0, 1)
    return np.clip(img, 0.0, 1.0)


def gaussian_noisy(clean: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """Unclipped additive Gaussian noise from the counter RNG (imaging.py:171-182)."""
    z = counter_normal(derive_seed(seed, 0x6E6F6973), clean.size, sigma).astype(np.float32)
    return (clean.astype(np.float32) + z.reshape(clean.shape)).astype(np.float32)


def microscopy_image(h: int, w: int, seed: int) -> np.ndarray:
    """Config 3: puncta + filaments, Poisson + read noise, normalised to [0,1]."""
    r = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    sig = np.full((h, w), 0.05)
    for _ in range(200):
        cy, cx, sg = r.uniform(0, h), r.uniform(0, w), r.uniform(1.5, 4.0)
        sig += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * sg * sg))
    for _ in range(30):
        pts = np.cumsum(r.normal(0, w / 12, size=(6, 2)), axis=0) + r.uniform(0, [h, w])
        for (y0, x0), (y1, x1) in zip(pts[:-1], pts[1:]):
            n = int(max(abs(y1 - y0), abs(x1 - x0))) + 1
            ys = np.clip(np.linspace(y0, y1, n).astype(int), 0, h - 2)
            xs = np.clip(np.linspace(x0, x1, n).astype(int), 0, w - 2)
            for dy in (0, 1):
                for dx in (0, 1):
                    sig[ys + dy, xs + dx] += 0.6
    photons = 30.0 * sig / sig.max()
    counts = r.poisson(photons).astype(np.float64) + r.normal(0, 2.0, size=(h, w))
    lo = counts.min()
    scale = (counts - lo).max()
    # the clean signal on the noisy image's scale (the expected counts through
    # the same affine normalisation), so PSNR compares like with like
    return ((counts - lo) / scale).astype(np.float32), ((photons - lo) / scale).astype(np.float32)


def config_image(cfg: int, seed: int = 0):
    """(noisy float32, clean float32) for BASELINE.json config 1/2/3/5 (4 = batch of 2)."""
    if cfg == 1:
        c = blob_rect_image(256, 256, seed)
        return gaussian_noisy(c, 25 / 255, seed + 1), c.astype(np.float32)
    if cfg in (2, 4):
        c = blob_rect_image(512, 512, seed)
        sigma = 50 / 255 if cfg == 2 else np.random.default_rng(seed + 7).uniform(15, 50) / 255
        return gaussian_noisy(c, sigma, seed + 1), c.astype(np.float32)
    if cfg == 3:
        return microscopy_image(1024, 1024, seed)
    if cfg == 5:
        c = blob_rect_image(4096, 4096, seed, n_blobs=400, n_rects=80)
        return gaussian_noisy(c, 25 / 255, seed + 1), c.astype(np.float32)
    raise ValueError(cfg)
