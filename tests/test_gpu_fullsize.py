"""Parity at BASELINE.json's full sizes (config 3: 1024^2 microscopy, config 5:
4096^2 blob+rectangle, config 4: a 512^2 member of the batch).

The NumPy oracle cannot run a network step at these sizes in test time, so:
  * integer/byte work (normalise, pair gather) is checked bit-exactly against
    the oracle at full size (NumPy gathers are fast);
  * the floating-point network work (one training step from the seeded init,
    the full-resolution validation forward) is checked against a PyTorch
    float64 / float32-without-TF32 restatement of the same network run on the
    GPU (the "plain PyTorch reference" the task allows for floating-point
    kernels), under the north_star bars: logits, gradients and updated
    parameters within 1e-3 norm-relative per layer;
  * size-independent properties of whole fits (determinism, finiteness, the
    window-mean identity, epoch accounting) through the public API.
"""

import ctypes as C

import numpy as np
import pytest

from n2f_testutil import arena_to_layers, norm_rel

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    assert torch.cuda.is_available()
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    return torch


def _engine(h, w, **cfg):
    from paper_2108_10209_b200 import Engine, TrainConfig

    return Engine(h, w, TrainConfig(**cfg), use_graph=False)


def _arena(eng, which):
    from paper_2108_10209_b200 import _lib

    n = C.c_int64()
    _lib.call("n2f_ctx_param_count", eng.handle, C.byref(n))
    out = np.empty(n.value, np.float32)
    _lib.call("n2f_ctx_get_arena", eng.handle, which, out.ctypes.data)
    return out


def _pairs(eng, h, w):
    from paper_2108_10209_b200 import _lib

    plane = h * (w // 2)
    pin, ptgt = np.empty(4 * plane, np.float32), np.empty(4 * plane, np.float32)
    norm = np.empty(h * w, np.float32)
    ph, pw = (C.c_int * 4)(), (C.c_int * 4)()
    _lib.call("n2f_ctx_get_pairs", eng.handle, pin.ctypes.data, ptgt.ctypes.data, norm.ctypes.data,
              ph, pw)
    pairs = []
    for k in range(4):
        n = ph[k] * pw[k]
        pairs.append((pin[k * plane: k * plane + n].reshape(ph[k], pw[k]),
                      ptgt[k * plane: k * plane + n].reshape(ph[k], pw[k])))
    return norm.reshape(h, w), pairs


def _torch_layers(torch, arena, shapes, dtype):
    return [(torch.tensor(w, dtype=dtype, device="cuda"), torch.tensor(b, dtype=dtype, device="cuda"))
            for w, b in arena_to_layers(arena, shapes)]


def _torch_forward(torch, layers, x):
    """model.py:72-90: 8 x (3x3 conv, zero pad 1, ReLU), then the 1x1 head."""
    F = torch.nn.functional
    last = len(layers) - 1
    for i, (w, b) in enumerate(layers):
        x = F.conv2d(x, w, b, padding=(w.shape[-1] - 1) // 2)
        if i != last:
            x = torch.relu(x)
    return x


def _predict_banded(torch, layers, norm, dtype, band=512):
    """Full-resolution validation forward in row bands with an 8-row halo (the
    receptive-field radius of the eight 3x3 layers), so a 4096^2 reference fits
    beside the engine's context; sigmoid + clip as model.py:123-140."""
    H, W = norm.shape
    halo = 8
    out = np.empty((H, W), np.float32)
    x_all = torch.tensor(norm, dtype=dtype, device="cuda")
    with torch.no_grad():
        for r0 in range(0, H, band):
            r1 = min(H, r0 + band)
            a0, a1 = max(0, r0 - halo), min(H, r1 + halo)
            z = _torch_forward(torch, layers, x_all[a0:a1][None, None])[0, 0]
            s = torch.sigmoid(z[r0 - a0: r0 - a0 + (r1 - r0)])
            out[r0:r1] = s.float().cpu().numpy()
    tiny = np.nextafter(np.float32(0), np.float32(1))
    return np.clip(out, tiny, np.nextafter(np.float32(1), np.float32(0)))


@pytest.fixture(scope="module")
def config3():
    from paper_2108_10209_b200 import synthetic

    noisy, clean = synthetic.config_image(3, 0)
    return noisy.astype(np.float64), clean


@pytest.fixture(scope="module")
def config5():
    from paper_2108_10209_b200 import synthetic

    noisy, clean = synthetic.config_image(5, 0)
    return noisy, clean


def _check_prep_bitwise(oracle, eng, img):
    norm64 = oracle.normalize(img)[0]
    n32 = norm64.astype(np.float32)
    norm, pairs = _pairs(eng, *img.shape)
    assert np.array_equal(norm, n32)
    for (a, b), (ra, rb) in zip(pairs, oracle.training_pairs(n32)):
        assert np.array_equal(a, ra) and np.array_equal(b, np.clip(rb, 0.0, 1.0))
    return n32, pairs


def test_config3_prep_step_and_validation(oracle, config3):
    """1024^2 microscopy image: bit-exact normalise/pairs/init, then the first
    training step (pair 0) and the validation pass after it against a float64
    PyTorch restatement (BCE mean loss, tensor.py:164-181; Adam t=1,
    tensor.py:125-141)."""
    from paper_2108_10209_b200 import _lib

    torch = _torch()
    img, _ = config3
    H, W = img.shape
    eng = _engine(H, W, seed=5)
    _lib.call("n2f_ctx_prepare", eng.handle, img.ctypes.data, _lib.N2F_F64, None, 1)
    n32, pairs = _check_prep_bitwise(oracle, eng, img)
    shapes = oracle.layer_shapes()
    p0 = _arena(eng, 0)
    from n2f_testutil import net_to_arena

    assert np.array_equal(p0, net_to_arena(oracle.init_net(5)))

    # engine step on pair 0
    a, t = pairs[0]
    z = np.empty(a.size, np.float32)
    _lib.call("n2f_ctx_step", eng.handle, 0, z.ctypes.data)
    grads = arena_to_layers(_arena(eng, 3), shapes)
    p1 = arena_to_layers(_arena(eng, 0), shapes)

    # float64 reference step
    f64 = torch.float64
    layers = _torch_layers(torch, p0, shapes, f64)
    for w, b in layers:
        w.requires_grad_(True)
        b.requires_grad_(True)
    x = torch.tensor(a, dtype=f64, device="cuda")[None, None]
    tt = torch.tensor(t, dtype=f64, device="cuda")
    zr = _torch_forward(torch, layers, x)[0, 0]
    loss = torch.nn.functional.binary_cross_entropy_with_logits(zr, tt)
    loss.backward()
    assert norm_rel(z, zr.detach().cpu().numpy().ravel()) < 1e-4
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    for li, ((w, b), (gw, gb), (ew, eb)) in enumerate(zip(layers, grads, p1)):
        rw, rb = w.grad.cpu().numpy(), b.grad.cpu().numpy()
        assert norm_rel(gw, rw) < 1e-3, ("grad w", li, norm_rel(gw, rw))
        assert norm_rel(gb, rb) < 1e-3, ("grad b", li, norm_rel(gb, rb))
        new = []
        for p, g in ((w, rw), (b, rb)):
            m = (1 - b1) * g
            v = (1 - b2) * g * g
            new.append(p.detach().cpu().numpy() - lr * (m / (1 - b1)) / (np.sqrt(v / (1 - b2)) + eps))
        err = norm_rel(np.concatenate([ew.ravel(), eb]), np.concatenate([new[0].ravel(), new[1]]))
        assert err < 1e-3, ("params", li, err)

    # validation pass with the engine's updated parameters
    out = np.empty(H * W, np.float32)
    score = C.c_double()
    _lib.call("n2f_ctx_validate", eng.handle, out.ctypes.data, C.byref(score))
    ref = _predict_banded(torch, _torch_layers(torch, _arena(eng, 0), shapes, f64), n32, f64)
    assert norm_rel(out.reshape(H, W), ref) < 1e-4
    assert abs(score.value - oracle.val_score(ref, n32)) < 1e-3 * score.value
    eng.close()


def test_config5_validation_pass_4096(oracle, config5):
    """4096^2: bit-exact normalise/pairs at full size, then the full-resolution
    validation forward (the HBM-heavy pass this config stresses) from the
    seeded init against a banded float32 (no TF32) PyTorch forward."""
    from paper_2108_10209_b200 import _lib

    torch = _torch()
    img, _ = config5
    H, W = img.shape
    eng = _engine(H, W, seed=9)
    _lib.call("n2f_ctx_prepare", eng.handle, img.ctypes.data, _lib.N2F_F32, None, 1)
    n32, _ = _check_prep_bitwise(oracle, eng, img)
    out = np.empty(H * W, np.float32)
    score = C.c_double()
    _lib.call("n2f_ctx_validate", eng.handle, out.ctypes.data, C.byref(score))
    assert np.isfinite(out).all()
    layers = _torch_layers(torch, _arena(eng, 0), oracle.layer_shapes(), torch.float32)
    ref = _predict_banded(torch, layers, n32, torch.float32)
    assert norm_rel(out.reshape(H, W), ref) < 1e-4
    assert abs(score.value - oracle.val_score(ref, n32)) < 1e-3 * score.value
    eng.close()
    del layers
    torch.cuda.empty_cache()


def test_config5_fit_epochs_4096(config5):
    """4096^2 through the public API: two epochs (max_epochs stop) with a
    two-slot window, finite output in the input's range, bitwise determinism
    of a repeated fit, and the window-mean identity: with window 1 the result
    is the last validation output, denormalised."""
    from paper_2108_10209_b200 import TrainConfig, train_single_channel
    from paper_2108_10209_b200 import trainer as T

    img, clean = config5
    cfg = TrainConfig(seed=2, max_epochs=2, patience_epochs=100, avg_window=2)
    a = train_single_channel(img, cfg)
    assert a.epochs_run == 2 and a.stop_reason == "max_epochs" and len(a.val_history) == 2
    assert a.denoised.shape == img.shape and a.denoised.dtype == np.float64
    assert np.isfinite(a.denoised).all()
    assert a.denoised.min() >= img.min() - 1e-6 and a.denoised.max() <= img.max() + 1e-6
    b = train_single_channel(img, cfg)
    assert np.array_equal(a.denoised, b.denoised) and a.val_history == b.val_history
    T.release_engines()


@pytest.mark.parametrize("seed", [3, 4])
def test_config4_member_window_identity(oracle, seed):
    """A config-4 image (512^2, per-image sigma U(15,50)/255): with a one-slot
    window the fit's result is exactly the denormalised last validation output
    (trainer.py:104-109, imaging.py:208-211); re-running validation on the
    fitted context reproduces that output bitwise."""
    from paper_2108_10209_b200 import _lib, synthetic

    noisy, _ = synthetic.config_image(4, seed)
    img = noisy.astype(np.float64)
    H, W = img.shape
    eng = _engine(H, W, seed=seed, max_epochs=3, avg_window=1, patience_epochs=100)
    out, r, hist, _, _ = eng.fit_host(np.ascontiguousarray(img))
    assert r.epochs_run == 3 and r.stop_reason == 1
    v = np.empty(H * W, np.float32)
    score = C.c_double()
    _lib.call("n2f_ctx_validate", eng.handle, v.ctypes.data, C.byref(score))
    assert abs(score.value - hist[-1]) <= 1e-12 * hist[-1]
    _, lo, hi, _ = oracle.normalize(img)
    expect = oracle.denormalize(v.reshape(H, W), lo, hi)
    assert np.array_equal(out, expect)
    eng.close()


def test_oversized_image_fails_cleanly_and_device_recovers():
    """Beyond one GPU's memory (a 12288^2 context needs ~700 GB): a clean
    error naming the allocation, nothing leaked, and the next fit works."""
    from paper_2108_10209_b200 import TrainConfig, _lib, synthetic, train_single_channel
    from paper_2108_10209_b200 import trainer as T

    T.release_engines()
    big = np.random.default_rng(0).random((12288, 12288), dtype=np.float32)
    with pytest.raises(_lib.N2FError, match="memory|cudaMalloc"):
        train_single_channel(big, TrainConfig(seed=0, max_epochs=1))
    del big
    clean = synthetic.blob_rect_image(64, 64, 2)
    img = synthetic.gaussian_noisy(clean, 25 / 255, 3).astype(np.float64)
    r = train_single_channel(img, TrainConfig(seed=0, max_epochs=2))
    assert r.epochs_run == 2 and np.isfinite(r.denoised).all()
    T.release_engines()
