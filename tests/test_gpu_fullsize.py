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


def _layers_arena(layers):
    """[(w_oihw, b)] (numpy) -> engine arena (K-major weights)."""
    from n2f_testutil import oihw_to_engine

    parts = []
    for w, b in layers:
        parts += [oihw_to_engine(np.asarray(w, np.float32)).ravel(), np.asarray(b, np.float32)]
    return np.ascontiguousarray(np.concatenate(parts), dtype=np.float32)


def _torch_grads(torch, layers, x, t, loss="bce"):
    """Manual backprop of model.py:92-113 with torch conv kernels, one layer at
    a time (only the post-ReLU activations are kept, so a 4096 x 2048 pair
    fits beside the engine's context).  Returns (logits, [(dW, db)])."""
    F = torch.nn.functional
    acts = [x]
    h = x
    last = len(layers) - 1
    with torch.no_grad():
        for i, (w, b) in enumerate(layers):
            h = F.conv2d(h, w, b, padding=(w.shape[-1] - 1) // 2)
            if i != last:
                h = torch.relu_(h)
            acts.append(h)
        z = acts.pop()[0, 0]
        n = z.numel()
        if loss == "bce":  # tensor.py:164-181: (sigmoid(z) - t) / N
            g = ((torch.sigmoid(z) - t) / n)[None, None]
        else:
            raise ValueError(loss)
        grads = [None] * len(layers)
        for i in range(last, -1, -1):
            w, b = layers[i]
            inp = acts.pop()
            pad = (w.shape[-1] - 1) // 2
            grads[i] = (torch.nn.grad.conv2d_weight(inp, w.shape, g, padding=pad), g.sum((0, 2, 3)))
            if i > 0:
                g = torch.nn.grad.conv2d_input(inp.shape, w, g, padding=pad) * (inp > 0)
            del inp
    return z, grads


def _adam_ref(p, g, m, v, t, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    """tensor.py:125-141 in float64."""
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    p = p - lr * (m / (1 - b1 ** t)) / (np.sqrt(v / (1 - b2 ** t)) + eps)
    return p, m, v


def test_config3_prep_and_all_four_steps(oracle, config3):
    """1024^2 microscopy image: bit-exact normalise/pairs/init, then ALL FOUR
    training steps of an epoch, each from an identical state on both sides
    (weights, Adam moments, t), against a float64 PyTorch restatement: logits
    < 1e-4, every layer's gradients and updated parameters < 1e-3
    norm-relative (north_star step bar); then the validation pass at the
    engine's end-of-epoch weights."""
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
    f64 = torch.float64
    # reference state (fp32 values, as both sides hold them), Adam moments zero
    P = [(w.astype(np.float64), b.astype(np.float64)) for w, b in arena_to_layers(p0, shapes)]
    M = [(np.zeros_like(w), np.zeros_like(b)) for w, b in P]
    V = [(np.zeros_like(w), np.zeros_like(b)) for w, b in P]
    for k, (a, t) in enumerate(pairs):
        r32 = lambda L: [(w.astype(np.float32), b.astype(np.float32)) for w, b in L]  # noqa: E731
        P, M, V = r32(P), r32(M), r32(V)
        for which, L in enumerate((P, M, V)):
            arr = _layers_arena(L)
            _lib.call("n2f_ctx_set_arena", eng.handle, which, arr.ctypes.data, k)
        z = np.empty(a.size, np.float32)
        _lib.call("n2f_ctx_step", eng.handle, k, z.ctypes.data)
        grads = arena_to_layers(_arena(eng, 3), shapes)
        got = arena_to_layers(_arena(eng, 0), shapes)
        layers = [(torch.tensor(w, dtype=f64, device="cuda"), torch.tensor(b, dtype=f64, device="cuda"))
                  for w, b in P]
        x = torch.tensor(a, dtype=f64, device="cuda")[None, None]
        tt = torch.tensor(t, dtype=f64, device="cuda")
        zr, rg = _torch_grads(torch, layers, x, tt)
        assert norm_rel(z, zr.cpu().numpy().ravel()) < 1e-4, ("logits", k)
        nP, nM, nV = [], [], []
        for li in range(len(shapes)):
            rw, rb = (q.cpu().numpy() for q in rg[li])
            gw, gb = grads[li]
            assert norm_rel(gw, rw) < 1e-3, ("grad w", k, li, norm_rel(gw, rw))
            assert norm_rel(gb, rb) < 1e-3, ("grad b", k, li, norm_rel(gb, rb))
            w1, mw, vw = _adam_ref(P[li][0].astype(np.float64), rw, M[li][0], V[li][0], k + 1)
            b1_, mb, vb = _adam_ref(P[li][1].astype(np.float64), rb, M[li][1], V[li][1], k + 1)
            ew, eb = got[li]
            err = norm_rel(np.concatenate([ew.ravel(), eb]), np.concatenate([w1.ravel(), b1_]))
            assert err < 1e-3, ("params", k, li, err)
            nP.append((w1, b1_))
            nM.append((mw, mb))
            nV.append((vw, vb))
        P, M, V = nP, nM, nV
        del layers, rg
    # validation pass with the engine's updated parameters (after step 4)
    out = np.empty(H * W, np.float32)
    score = C.c_double()
    _lib.call("n2f_ctx_validate", eng.handle, out.ctypes.data, C.byref(score))
    ref = _predict_banded(torch, _torch_layers(torch, _arena(eng, 0), shapes, f64), n32, f64)
    assert norm_rel(out.reshape(H, W), ref) < 1e-4
    assert abs(score.value - oracle.val_score(ref, n32)) < 1e-3 * score.value
    eng.close()
    torch.cuda.empty_cache()


def test_config5_training_step_4096(oracle, config5):
    """4096^2 (config 5): one training step (pair 0, a 4096 x 2048 plane) from
    the seeded init against a float32 (TF32 off) PyTorch restatement run beside
    the engine's ~79 GiB context: logits < 1e-4, every layer's gradients and
    updated parameters < 1e-3 norm-relative."""
    from paper_2108_10209_b200 import _lib

    torch = _torch()
    img, _ = config5
    H, W = img.shape
    eng = _engine(H, W, seed=9)
    _lib.call("n2f_ctx_prepare", eng.handle, img.ctypes.data, _lib.N2F_F32, None, 1)
    shapes = oracle.layer_shapes()
    p0 = _arena(eng, 0)
    norm, pairs = _pairs(eng, H, W)
    a, t = pairs[0]
    z = np.empty(a.size, np.float32)
    _lib.call("n2f_ctx_step", eng.handle, 0, z.ctypes.data)
    grads = arena_to_layers(_arena(eng, 3), shapes)
    got = arena_to_layers(_arena(eng, 0), shapes)
    f32 = torch.float32
    layers = _torch_layers(torch, p0, shapes, f32)
    zr, rg = _torch_grads(torch, layers, torch.tensor(a, device="cuda")[None, None],
                          torch.tensor(t, device="cuda"))
    assert norm_rel(z, zr.cpu().numpy().ravel()) < 1e-4
    for li, (w0, b0) in enumerate(arena_to_layers(p0, shapes)):
        rw, rb = (q.double().cpu().numpy() for q in rg[li])
        gw, gb = grads[li]
        assert norm_rel(gw, rw) < 1e-3, ("grad w", li, norm_rel(gw, rw))
        assert norm_rel(gb, rb) < 1e-3, ("grad b", li, norm_rel(gb, rb))
        w1 = _adam_ref(w0.astype(np.float64), rw, 0.0, 0.0, 1)[0]
        b1_ = _adam_ref(b0.astype(np.float64), rb, 0.0, 0.0, 1)[0]
        ew, eb = got[li]
        err = norm_rel(np.concatenate([ew.ravel(), eb]), np.concatenate([w1.ravel(), b1_]))
        assert err < 1e-3, ("params", li, err)
    del layers, rg, zr
    torch.cuda.empty_cache()
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
