"""Shared helpers for the GPU parity tests: device buffers via torch, layout
permutations between the oracle (OIHW / CHW) and the engine (K-major / HWC)."""

from __future__ import annotations

import numpy as np


def torch_cuda():
    import torch

    assert torch.cuda.is_available(), "GPU test needs CUDA"
    return torch


def dev(a: np.ndarray):
    torch = torch_cuda()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t) -> np.ndarray:
    return t.detach().cpu().numpy()


def empty(shape, dtype=np.float32):
    torch = torch_cuda()
    tdt = {np.float32: torch.float32, np.float64: torch.float64}[np.dtype(dtype).type]
    return torch.empty(shape, dtype=tdt, device="cuda")


def oihw_to_engine(w: np.ndarray) -> np.ndarray:
    """(cout, cin, kh, kw) -> (cout, kh, kw, cin)."""
    return np.ascontiguousarray(w.transpose(0, 2, 3, 1))


def engine_to_oihw(w: np.ndarray, cout: int, cin: int, k: int) -> np.ndarray:
    return np.ascontiguousarray(w.reshape(cout, k, k, cin).transpose(0, 3, 1, 2))


def chw_to_hwc(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x.transpose(1, 2, 0))


def hwc_to_chw(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x.transpose(2, 0, 1))


def net_to_arena(net) -> np.ndarray:
    parts = []
    for w, b in zip(net.weights, net.biases):
        parts += [oihw_to_engine(w).reshape(-1), b.reshape(-1)]
    return np.concatenate(parts).astype(np.float32)


def arena_to_layers(arena: np.ndarray, shapes):
    """Split an engine arena into [(w_oihw, b)] for the oracle's layer shapes."""
    out, off = [], 0
    for cin, cout, k in shapes:
        n = cout * k * k * cin
        w = engine_to_oihw(arena[off: off + n], cout, cin, k)
        off += n
        b = arena[off: off + cout].copy()
        off += cout
        out.append((w, b))
    assert off == arena.size
    return out


def norm_rel(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def psnr(a, b, data_range=1.0) -> float:
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(data_range * data_range / mse)
