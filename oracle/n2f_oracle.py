"""CPU oracle for the Noise2Fast fit-and-denoise path -- TEST INFRASTRUCTURE ONLY.

This module is a plain NumPy restatement of the reference package's hot path
(`/root/reference/pkg/src/noise2fast`, cited per function below).  It exists
so that the parity tests, ``__graft_entry__.smoke()`` and the ``cpu_baseline``
leg of ``bench.py`` have a checker that travels to the GPU box (the reference
tree does not).  Nothing in the product package may import it: the product
path runs only through the CUDA C-ABI library and fails loudly without it.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
fixtures in ``tests/golden/`` that were produced by importing the real
reference (``tests/golden/make_golden.py``); bit-exact where the reference is
deterministic integer/byte/IEEE work (RNG, init, normalize, downsample, Adam,
stop rule, window mean) and within fp32 reassociation tolerance for the
BLAS-backed convolutions.

Array conventions: single images are 2-D ``(h, w)``; feature maps are
``(c, h, w)`` float32 (batch 1 is implicit).  Conv weights are OIHW float32 as
in the reference (`tensor.py:75-105`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# counter RNG  (rng.py:14-78)
# --------------------------------------------------------------------------

_M64 = 0xFFFFFFFFFFFFFFFF
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix_finalize(words: np.ndarray) -> np.ndarray:
    """SplitMix64 output function on uint64 words (rng.py:20-28)."""
    z = np.asarray(words, dtype=np.uint64) + _GAMMA
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def child_seed(seed: int, *ids: int) -> int:
    """Fold stream ids into a seed (rng.py:31-39)."""
    acc = np.uint64(seed & _M64)
    for i in ids:
        acc = splitmix_finalize(np.array([acc ^ np.uint64(i & _M64)], dtype=np.uint64))[0]
    return int(acc)


def counter_uniform(seed: int, n: int, low: float, high: float, start: int = 0) -> np.ndarray:
    """Doubles in [low, high) from counter slots start..start+n (rng.py:52-64)."""
    key = splitmix_finalize(np.array([seed & _M64], dtype=np.uint64))[0]
    ctr = np.arange(start, start + n, dtype=np.uint64)
    bits = splitmix_finalize(ctr ^ key)
    u = (bits >> np.uint64(11)).astype(np.float64) * float(2.0**-53)
    return low + u * (high - low)


def counter_normal(seed: int, n: int, sigma: float = 1.0) -> np.ndarray:
    """Box-Muller normals on 53-bit uniforms (rng.py:66-78)."""
    half = (n + 1) // 2
    key = splitmix_finalize(np.array([seed & _M64], dtype=np.uint64))[0]
    bits = splitmix_finalize(np.arange(0, 2 * half, dtype=np.uint64) ^ key)
    u = (bits >> np.uint64(11)).astype(np.float64) * float(2.0**-53)
    rad = np.sqrt(-2.0 * np.log(1.0 - u[:half]))
    ang = 2.0 * np.pi * u[half:]
    return np.concatenate([rad * np.cos(ang), rad * np.sin(ang)])[:n] * sigma


# --------------------------------------------------------------------------
# network definition and init  (model.py:20, 36-65)
# --------------------------------------------------------------------------

WIDTHS = (32, 32, 64, 64, 128, 128, 256, 256)


def layer_shapes(in_ch: int = 1):
    """(cin, cout, k) for the 8 3x3 ReLU layers then the 1x1 head."""
    shapes, prev = [], in_ch
    for c in WIDTHS:
        shapes.append((prev, c, 3))
        prev = c
    shapes.append((prev, 1, 1))
    return shapes


@dataclass
class OracleNet:
    weights: list  # OIHW float32
    biases: list  # (cout,) float32
    m: list = field(default_factory=list)  # Adam first moments, [w0,b0,w1,b1,...]
    v: list = field(default_factory=list)
    t: int = 0


def init_net(seed: int, in_ch: int = 1) -> OracleNet:
    """He-uniform init from per-layer counter streams (model.py:46-65)."""
    ws, bs = [], []
    for idx, (cin, cout, k) in enumerate(layer_shapes(in_ch)):
        fan_in = cin * k * k
        b = math.sqrt(6.0 / fan_in)
        vals = counter_uniform(child_seed(seed, idx), cout * fan_in, -b, b)
        ws.append(vals.astype(np.float32).reshape(cout, cin, k, k))
        bs.append(np.zeros(cout, dtype=np.float32))
    net = OracleNet(ws, bs)
    for w, bb in zip(ws, bs):
        net.m += [np.zeros_like(w), np.zeros_like(bb)]
        net.v += [np.zeros_like(w), np.zeros_like(bb)]
    return net


def params_flat(net: OracleNet):
    out = []
    for w, b in zip(net.weights, net.biases):
        out += [w, b]
    return out


# --------------------------------------------------------------------------
# normalisation, downsampling  (imaging.py:190-211, downsample.py:45-164)
# --------------------------------------------------------------------------


def normalize(img: np.ndarray):
    """(x-min)/(max-min) in f64; returns (norm f64, vmin, vmax, degenerate)."""
    x = np.asarray(img, dtype=np.float64)
    lo, hi = float(x.min()), float(x.max())
    if lo == hi:
        return np.full(x.shape, 0.5), lo, hi, True
    return (x - lo) / (hi - lo), lo, hi, False


def denormalize(plane: np.ndarray, lo: float, hi: float) -> np.ndarray:
    return np.asarray(plane, dtype=np.float64) * (hi - lo) + lo


def even_crop(x: np.ndarray) -> np.ndarray:
    h, w = x.shape
    return x[: h & ~1, : w & ~1]


def checkerboard(x: np.ndarray):
    """Four checkerboard compactions (eu, ou, el, ol) (downsample.py:45-66).

    eu[i,j] = x[i, 2j+(i&1)]       ou[i,j] = x[i, 2j+1-(i&1)]
    el[i,j] = x[2i+(j&1), j]       ol[i,j] = x[2i+1-(j&1), j]
    """
    h, w = x.shape
    assert h % 2 == 0 and w % 2 == 0
    rows = np.arange(h)[:, None]
    cols2 = 2 * np.arange(w // 2)[None, :]
    eu = x[rows, cols2 + (rows & 1)]
    ou = x[rows, cols2 + 1 - (rows & 1)]
    rows2 = 2 * np.arange(h // 2)[:, None]
    cols = np.arange(w)[None, :]
    el = x[rows2 + (cols & 1), cols]
    ol = x[rows2 + 1 - (cols & 1), cols]
    return eu, ou, el, ol


def quad_phases(x: np.ndarray):
    """2x2-block phase images (TL, TR, BL, BR) (downsample.py:94-100)."""
    return x[0::2, 0::2], x[0::2, 1::2], x[1::2, 0::2], x[1::2, 1::2]


def training_pairs(norm32: np.ndarray, scheme: str = "checkerboard", clean32=None):
    """Fixed-order (input, target) list (downsample.py:110-164, trainer.py:164-176)."""
    x = even_crop(norm32)
    if scheme == "checkerboard":
        eu, ou, el, ol = checkerboard(x)
        return [(eu, ou), (ou, eu), (el, ol), (ol, el)]
    if scheme == "quad":
        tl, tr, bl, _ = quad_phases(x)
        return [(tl, tr), (tr, tl), (tl, bl), (bl, tl)]
    if scheme == "exact":
        s = even_crop(clean32)
        xe = checkerboard(x)
        se = checkerboard(s)
        out = []
        for a, b in ((0, 1), (1, 0), (2, 3), (3, 2)):
            out.append((xe[a], xe[b] - (se[b] - se[a])))
        return out
    raise ValueError(scheme)


# --------------------------------------------------------------------------
# fp32 convolution via im2col + GEMM  (tensor.py:231-316, 490-530)
# --------------------------------------------------------------------------


def _patches(x: np.ndarray, k: int) -> np.ndarray:
    """(c, h, w) -> (c*k*k, h*w) with zero padding (k-1)/2."""
    c, h, w = x.shape
    if k == 1:
        return x.reshape(c, h * w)
    p = k // 2
    xp = np.zeros((c, h + 2 * p, w + 2 * p), dtype=x.dtype)
    xp[:, p : p + h, p : p + w] = x
    cols = np.empty((c, k, k, h, w), dtype=x.dtype)
    for dy in range(k):
        for dx in range(k):
            cols[:, dy, dx] = xp[:, dy : dy + h, dx : dx + w]
    return cols.reshape(c * k * k, h * w)


def conv_forward(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Pre-activation of one same-size conv; x (cin,h,w) -> (cout,h,w)."""
    cout, cin, k, _ = w.shape
    _, h, wd = x.shape
    pre = np.matmul(w.reshape(cout, -1), _patches(x, k))
    pre += b[:, None]
    return pre.reshape(cout, h, wd)


def conv_backward(gpre: np.ndarray, x: np.ndarray, w: np.ndarray, need_dx: bool):
    """(dx, dw, db) given the gradient at the pre-activation."""
    cout, cin, k, _ = w.shape
    _, h, wd = x.shape
    g = gpre.reshape(cout, h * wd)
    db = g.sum(axis=1)
    cols = _patches(x, k)
    dw = np.matmul(g, cols.T).reshape(w.shape)
    dx = None
    if need_dx:
        gc = np.matmul(w.reshape(cout, -1).T, g)
        if k == 1:
            dx = gc.reshape(cin, h, wd)
        else:
            p = k // 2
            acc = np.zeros((cin, h + 2 * p, wd + 2 * p), dtype=x.dtype)
            gc = gc.reshape(cin, k, k, h, wd)
            for dy in range(k):
                for dx_ in range(k):
                    acc[:, dy : dy + h, dx_ : dx_ + wd] += gc[:, dy, dx_]
            dx = np.ascontiguousarray(acc[:, p : p + h, p : p + wd])
    return dx, dw, db


# --------------------------------------------------------------------------
# activations, losses, optimizer  (tensor.py:108-193)
# --------------------------------------------------------------------------


def sigmoid(z: np.ndarray) -> np.ndarray:
    """Two-branch logistic (tensor.py:153-161)."""
    out = np.empty_like(z)
    nonneg = z >= 0
    out[nonneg] = 1.0 / (1.0 + np.exp(-z[nonneg]))
    e = np.exp(z[~nonneg])
    out[~nonneg] = e / (1.0 + e)
    return out


def bce_logits(z: np.ndarray, t: np.ndarray):
    """(mean loss, dloss/dz) for sigmoid+BCE (tensor.py:164-181)."""
    per = np.maximum(z, 0) - z * t + np.log1p(np.exp(-np.abs(z)))
    grad = (sigmoid(z) - t) / z.size
    return float(per.mean()), grad.astype(z.dtype, copy=False)


def mse_sigmoid(z: np.ndarray, t: np.ndarray):
    """MSE through the sigmoid (trainer.py:112-117, tensor.py:184-193)."""
    s = sigmoid(z)
    d = s - t
    loss = float(np.mean(d * d))
    gs = ((2.0 / s.size) * d).astype(s.dtype, copy=False)
    return loss, gs * s * (1 - s)


BETA1, BETA2, EPS = 0.9, 0.999, 1e-8


def adam_update(p: np.ndarray, g: np.ndarray, m: np.ndarray, v: np.ndarray, t: int, lr: float):
    """In-place Adam with NumPy-2 weak-scalar fp32 semantics (tensor.py:125-141)."""
    m *= BETA1
    m += (1.0 - BETA1) * g
    v *= BETA2
    v += (1.0 - BETA2) * (g * g)
    mh = m / (1.0 - BETA1**t)
    vh = v / (1.0 - BETA2**t)
    p -= lr * mh / (np.sqrt(vh) + EPS)


# --------------------------------------------------------------------------
# network passes  (model.py:72-140)
# --------------------------------------------------------------------------


def net_forward(net: OracleNet, img: np.ndarray, keep: bool):
    """Logits (h,w) plus, when keep, [(layer input, pre-activation)]."""
    x = img[None].astype(np.float32, copy=False)
    cache = []
    last = len(net.weights) - 1
    for i, (w, b) in enumerate(zip(net.weights, net.biases)):
        pre = conv_forward(x, w, b)
        if keep:
            cache.append((x, pre))
        x = pre if i == last else np.maximum(pre, 0)
    return x[0], cache


def net_backward(net: OracleNet, cache, gz: np.ndarray):
    grads = [None] * len(net.weights)
    g = gz[None]
    last = len(net.weights) - 1
    for i in range(last, -1, -1):
        x, pre = cache[i]
        gp = g if i == last else g * (pre > 0)
        g, dw, db = conv_backward(gp, x, net.weights[i], need_dx=i > 0)
        grads[i] = (dw, db)
    return grads


def net_step(net: OracleNet, grads, lr: float):
    net.t += 1
    k = 0
    for i in range(len(net.weights)):
        for p, g in ((net.weights[i], grads[i][0]), (net.biases[i], grads[i][1])):
            adam_update(p, g, net.m[k], net.v[k], net.t, lr)
            k += 1


TINY32 = np.nextafter(np.float32(0), np.float32(1))
TOP32 = np.nextafter(np.float32(1), np.float32(0))


def predict(net: OracleNet, norm32: np.ndarray) -> np.ndarray:
    z, _ = net_forward(net, norm32, keep=False)
    return np.clip(sigmoid(z), TINY32, TOP32)


def val_score(out32: np.ndarray, norm32: np.ndarray) -> float:
    """f64 MSE of the output against the noisy input (trainer.py:97-101)."""
    d = out32.astype(np.float64) - norm32.astype(np.float64)
    return float(np.mean(d * d))


# --------------------------------------------------------------------------
# protocol: stop rule, window mean, full loop  (trainer.py:54-213)
# --------------------------------------------------------------------------


class StopTracker:
    """Strict-improvement patience counter plus output ring (trainer.py:78-94)."""

    def __init__(self, patience: int, window: int):
        self.patience, self.window = patience, window
        self.best = math.inf
        self.since = 0
        self.epoch = 0
        self.history: list[float] = []
        self.ring: list[np.ndarray] = []

    def push(self, score: float, out: np.ndarray) -> bool:
        self.epoch += 1
        self.history.append(score)
        self.ring.append(out)
        if len(self.ring) > self.window:
            self.ring.pop(0)
        if score < self.best:
            self.best, self.since = score, 0
        else:
            self.since += 1
        return self.since >= self.patience


def window_mean(outs) -> np.ndarray:
    """Sequential fp32 sum in epoch order divided by n (trainer.py:104-109)."""
    acc = outs[0].astype(np.float32).copy()
    for o in outs[1:]:
        acc += o
    return (acc / np.float32(len(outs))).astype(np.float32)


@dataclass
class OracleResult:
    denoised: np.ndarray
    epochs_run: int
    val_history: list
    stop_reason: str
    train_losses: list


def fit_denoise(noisy, *, seed=0, lr=1e-3, patience=100, window=100, max_epochs=20000,
                loss="bce", scheme="checkerboard", clean=None, net: OracleNet | None = None):
    """The whole per-image loop (trainer.py:125-213)."""
    x = np.asarray(noisy, dtype=np.float64)
    norm, lo, hi, degen = normalize(x)
    if degen:
        return OracleResult(x.copy(), 0, [], "degenerate", [])
    n32 = norm.astype(np.float32)
    c32 = None
    if scheme == "exact":
        c32 = ((np.asarray(clean, dtype=np.float64) - lo) / (hi - lo)).astype(np.float32)
    pairs = training_pairs(n32, scheme, c32)
    if loss == "bce":
        pairs = [(a, np.clip(b, 0.0, 1.0)) for a, b in pairs]
    net = net or init_net(seed)
    tracker = StopTracker(patience, window)
    reason, losses = "max_epochs", []
    for _ in range(max_epochs):
        ep = []
        for a, b in pairs:
            z, cache = net_forward(net, a, keep=True)
            lv, gz = bce_logits(z, b) if loss == "bce" else mse_sigmoid(z, b)
            net_step(net, net_backward(net, cache, gz), lr)
            ep.append(lv)
        losses.append(ep)
        out = predict(net, n32)
        if tracker.push(val_score(out, n32), out):
            reason = "patience"
            break
    den = denormalize(window_mean(tracker.ring), lo, hi)
    return OracleResult(den, tracker.epoch, tracker.history, reason, losses)


# --------------------------------------------------------------------------
# image-quality metrics  (imaging.py:249-311; benchmark mode)
# --------------------------------------------------------------------------


def psnr(a, b, data_range: float) -> float:
    """10 log10(range^2 / MSE) in f64, +inf for identical inputs (imaging.py:249-263)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    mse = float(np.mean((a - b) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(data_range * data_range / mse)


def gaussian_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    """Normalised 1-D Gaussian taps (imaging.py:266-270)."""
    coords = np.arange(size) - (size - 1) / 2.0
    g = np.exp(-(coords ** 2) / (2.0 * sigma * sigma))
    return g / g.sum()


def _valid_window_mean(x: np.ndarray, win: np.ndarray) -> np.ndarray:
    """Separable weighted window sums over fully valid positions: rows first,
    then columns (imaging.py:273-278 correlates with zero padding and crops the
    border, which leaves exactly these positions)."""
    k = win.size
    h, w = x.shape
    y = sum(win[i] * x[i: h - k + 1 + i, :] for i in range(k))
    return sum(win[j] * y[:, j: w - k + 1 + j] for j in range(k))


def ssim(a, b, data_range: float, k1: float = 0.01, k2: float = 0.03) -> float:
    """Mean SSIM with the 11x11 Gaussian window (imaging.py:281-311)."""
    a = np.squeeze(np.asarray(a, dtype=np.float64))
    b = np.squeeze(np.asarray(b, dtype=np.float64))
    win = gaussian_window()
    mu_a = _valid_window_mean(a, win)
    mu_b = _valid_window_mean(b, win)
    var_a = _valid_window_mean(a * a, win) - mu_a * mu_a
    var_b = _valid_window_mean(b * b, win) - mu_b * mu_b
    cov = _valid_window_mean(a * b, win) - mu_a * mu_b
    c1 = (k1 * data_range) ** 2
    c2 = (k2 * data_range) ** 2
    num = (2 * mu_a * mu_b + c1) * (2 * cov + c2)
    den = (mu_a ** 2 + mu_b ** 2 + c1) * (var_a + var_b + c2)
    return float(np.mean(num / den))
