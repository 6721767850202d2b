"""Image-quality metrics on the device: drop-ins for the reference's
``imaging.psnr`` and ``imaging.ssim`` (imaging.py:249-311), used by its
benchmark mode (cli.py:113-139).

Both take arrays (or objects with a ``samples`` attribute, like the
reference's ImageData) and compute in f64 exactly like the reference: PSNR =
10 log10(range^2 / MSE) (+inf for identical inputs); SSIM = mean over the
fully valid positions of the 11x11 Gaussian-window (sigma 1.5) structural
similarity.  The arithmetic runs in libn2f's kernels (``n2f_psnr``,
``n2f_ssim``); there is no CPU fallback.  CUDA tensors are used in place.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _samples(x):
    return x.samples if hasattr(x, "samples") else x


def _device_f64(x):
    """(tensor on the current CUDA device as contiguous f64, numpy-like shape)."""
    import torch

    if isinstance(x, torch.Tensor):
        t = x.detach()
        if not t.is_cuda:
            t = t.cuda()
        return t.to(torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=np.float64)).cuda()


def _shape(x):
    return tuple(x.shape)


def psnr(a, b, data_range: float) -> float:
    """Peak signal-to-noise ratio in dB (imaging.py:249-263)."""
    a, b = _samples(a), _samples(b)
    if _shape(a) != _shape(b):
        raise ValueError(f"shape mismatch: {_shape(a)} vs {_shape(b)}")
    if data_range <= 0:
        raise ValueError("data_range must be positive")
    da, db = _device_f64(a), _device_f64(b)
    out = C.c_double()
    _lib.call("n2f_psnr", da.data_ptr(), db.data_ptr(), da.numel(), float(data_range), C.byref(out),
              None)
    return float(out.value)


def ssim(a, b, data_range: float, k1: float = 0.01, k2: float = 0.03) -> float:
    """Mean SSIM, 11x11 Gaussian window, valid positions (imaging.py:266-311)."""
    a, b = _samples(a), _samples(b)
    sa = tuple(d for d in _shape(a) if d != 1)
    sb = tuple(d for d in _shape(b) if d != 1)
    if sa != sb:
        raise ValueError(f"shape mismatch: {sa} vs {sb}")
    if len(sa) != 2:
        raise ValueError("ssim expects a single-channel 2-D image per call")
    if min(sa) < 11:
        raise ValueError(f"image {sa} smaller than the 11x11 window")
    if data_range <= 0:
        raise ValueError("data_range must be positive")
    da, db = _device_f64(a), _device_f64(b)
    out = C.c_double()
    _lib.call("n2f_ssim", da.data_ptr(), db.data_ptr(), sa[0], sa[1], float(data_range), float(k1),
              float(k2), C.byref(out), None)
    return float(out.value)
