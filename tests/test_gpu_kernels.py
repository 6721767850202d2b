"""Per-kernel parity: the CUDA kernels (through the C ABI) vs the CPU oracle.

Bit-exact for the integer/IEEE-ordered work (normalise, pair gather, init,
Adam, stop rule, window mean); fp32 reassociation tolerance for the
convolutions (the reference's own 1e-5-of-scale bar, test_tensor.py:82-88)
and for the transcendental loss/sigmoid (GPU expf vs NumPy exp).
"""

import ctypes as C

import numpy as np
import pytest

from n2f_testutil import (chw_to_hwc, dev, empty, engine_to_oihw, host, hwc_to_chw,
                          oihw_to_engine)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2108_10209_b200 import _lib

    return _lib


def _call(lib, name, *args):
    lib.call(name, *args)


@pytest.mark.parametrize("hw", [(4, 4), (7, 9), (13, 17), (64, 48), (33, 130), (512, 512)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("scheme", [0, 1, 2])
def test_normalize_and_pairs_bitwise(lib, oracle, hw, dtype, scheme):
    rng = np.random.default_rng(hash((hw, scheme)) % 2**32)
    img = (rng.normal(0.3, 1.7, hw)).astype(dtype)
    clean = (rng.normal(0.2, 1.0, hw)).astype(dtype)
    d_img, d_clean = dev(img), dev(clean)
    mm = np.zeros(3)
    code = lib.N2F_F64 if dtype == np.float64 else lib.N2F_F32
    _call(lib, "n2f_minmax", d_img.data_ptr(), code, img.size, mm.ctypes.data, None)
    norm64, lo, hi, _ = oracle.normalize(img)
    assert mm[0] == lo and mm[1] == hi and mm[2] == 0
    He, We = hw[0] & ~1, hw[1] & ~1
    plane = (He // 2) * (We // 2) if scheme == 1 else He * (We // 2)
    d_norm = empty(img.size)
    d_in, d_tgt = empty(4 * plane), empty(4 * plane)
    ph, pw = (C.c_int * 4)(), (C.c_int * 4)()
    _call(lib, "n2f_make_pairs", d_img.data_ptr(), code, d_clean.data_ptr(), hw[0], hw[1], lo, hi,
          scheme, 1, d_norm.data_ptr(), d_in.data_ptr(), d_tgt.data_ptr(), ph, pw, None)
    n32 = norm64.astype(np.float32)
    assert np.array_equal(host(d_norm).reshape(hw), n32)
    c32 = ((clean.astype(np.float64) - lo) / (hi - lo)).astype(np.float32)
    pairs = oracle.training_pairs(n32, ["checkerboard", "quad", "exact"][scheme], c32)
    gin, gtgt = host(d_in), host(d_tgt)
    for k, (a, b) in enumerate(pairs):
        assert (ph[k], pw[k]) == a.shape
        got_a = gin[k * plane: k * plane + a.size].reshape(a.shape)
        got_b = gtgt[k * plane: k * plane + b.size].reshape(b.shape)
        assert np.array_equal(got_a, a), k
        assert np.array_equal(got_b, np.clip(b, 0.0, 1.0)), k


def test_minmax_flags_nonfinite(lib):
    img = np.ones((8, 8), np.float32)
    img[3, 4] = np.nan
    img[0, 0] = np.inf
    mm = np.zeros(3)
    d_img = dev(img)
    _call(lib, "n2f_minmax", d_img.data_ptr(), lib.N2F_F32, img.size, mm.ctypes.data, None)
    assert mm[2] == 2


@pytest.mark.parametrize("seed", [0, 7, 4242, 2**64 - 3])
def test_init_bitwise(lib, oracle, seed):
    net = oracle.init_net(seed)
    for li, (cin, cout, k) in enumerate(oracle.layer_shapes()):
        d = empty(cout * k * k * cin)
        _call(lib, "n2f_init_layer", seed, li, cin, cout, k, d.data_ptr(), None)
        got = engine_to_oihw(host(d), cout, cin, k)
        assert np.array_equal(got, net.weights[li]), li


CONV_SHAPES = [(1, 32, 3), (32, 32, 3), (32, 64, 3), (64, 64, 3), (64, 128, 3), (128, 128, 3),
               (128, 256, 3), (256, 256, 3), (256, 1, 1)]


IMPL = 3  # tcgen05 FP16x3, the library's only conv implementation (L1 / the 1x1 head:
          # the first-layer and head kernels)


@pytest.mark.parametrize("cin,cout,k", CONV_SHAPES)
@pytest.mark.parametrize("hw", [(13, 17), (40, 24), (64, 96)])
def test_conv_forward(lib, oracle, cin, cout, k, hw):
    impl = IMPL
    rng = np.random.default_rng(cin * 1000 + cout + hw[0])
    x = rng.standard_normal((cin, *hw)).astype(np.float32)
    w = (rng.standard_normal((cout, cin, k, k)) / np.sqrt(cin * k * k)).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    pre = oracle.conv_forward(x, w, b)
    for relu in (0, 1):
        ref = np.maximum(pre, 0) if relu else pre
        y = empty(hw[0] * hw[1] * cout)
        d_x, d_w, d_b = dev(chw_to_hwc(x)), dev(oihw_to_engine(w)), dev(b)  # keep alive
        _call(lib, "n2f_conv_fwd", d_x.data_ptr(), d_w.data_ptr(), d_b.data_ptr(), y.data_ptr(),
              hw[0], hw[1], cin, cout, k, relu, impl, None)
        got = hwc_to_chw(host(y).reshape(*hw, cout))
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-5 * np.abs(ref).max())


@pytest.mark.parametrize("cin,cout,k", CONV_SHAPES)
@pytest.mark.parametrize("hw", [(13, 17), (40, 24), (64, 96)])
def test_conv_backward(lib, oracle, cin, cout, k, hw):
    impl = IMPL
    rng = np.random.default_rng(cin * 77 + cout + hw[1])
    x = np.maximum(rng.standard_normal((cin, *hw)), 0).astype(np.float32)  # post-ReLU input
    w = (rng.standard_normal((cout, cin, k, k)) / np.sqrt(cin * k * k)).astype(np.float32)
    g = rng.standard_normal((cout, *hw)).astype(np.float32)
    dx_ref, dw_ref, db_ref = oracle.conv_backward(g, x, w, need_dx=True)
    dx_ref = dx_ref * (x > 0)  # the engine fuses the previous layer's ReLU mask
    P = hw[0] * hw[1]
    d_x = dev(chw_to_hwc(x))
    d_dw, d_db = empty(w.size), empty(cout)
    need_dx = cin > 1
    d_dx = empty(P * cin) if need_dx else None
    d_g, d_w = dev(chw_to_hwc(g)), dev(oihw_to_engine(w))
    _call(lib, "n2f_conv_bwd", d_g.data_ptr(), d_x.data_ptr(),
          d_w.data_ptr(), d_x.data_ptr() if need_dx else None,
          d_dx.data_ptr() if need_dx else None, d_dw.data_ptr(), d_db.data_ptr(), hw[0], hw[1],
          cin, cout, k, impl, None)
    dw = engine_to_oihw(host(d_dw), cout, cin, k)
    np.testing.assert_allclose(dw, dw_ref, rtol=0, atol=1e-5 * np.abs(dw_ref).max())
    np.testing.assert_allclose(host(d_db), db_ref, rtol=0, atol=1e-5 * np.abs(db_ref).max())
    if need_dx:
        dx = hwc_to_chw(host(d_dx).reshape(*hw, cin))
        np.testing.assert_allclose(dx, dx_ref, rtol=0, atol=1e-5 * np.abs(dx_ref).max())


def _random_conv_cases(n, seed):
    """Seeded random (layer shape, image size) cases in the spirit of the
    reference's 200-shape acceptance sweep (test_acceptance.py:183-229): every
    layer shape of the network over ragged sizes from 1 pixel to a few tile
    rows / columns, including 1 x W and H x 1 planes."""
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(n):
        cin, cout, k = CONV_SHAPES[i % len(CONV_SHAPES)]
        h, w = int(rng.integers(1, 41)), int(rng.integers(1, 71))
        if i % 7 == 0:
            h = 1
        if i % 11 == 0:
            w = 1
        cases.append((cin, cout, k, h, w))
    return cases


@pytest.mark.parametrize("cin,cout,k,h,w", _random_conv_cases(45, 2108))
def test_conv_forward_backward_random_shapes(lib, oracle, cin, cout, k, h, w):
    rng = np.random.default_rng(cin * 31 + cout * 7 + h * 131 + w)
    x = np.maximum(rng.standard_normal((cin, h, w)), 0).astype(np.float32)
    wt = (rng.standard_normal((cout, cin, k, k)) / np.sqrt(cin * k * k)).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    g = rng.standard_normal((cout, h, w)).astype(np.float32)
    P = h * w
    d_x, d_w, d_b, d_g = dev(chw_to_hwc(x)), dev(oihw_to_engine(wt)), dev(b), dev(chw_to_hwc(g))
    y = empty(P * cout)
    _call(lib, "n2f_conv_fwd", d_x.data_ptr(), d_w.data_ptr(), d_b.data_ptr(), y.data_ptr(),
          h, w, cin, cout, k, 1, IMPL, None)
    ref = np.maximum(oracle.conv_forward(x, wt, b), 0)
    got = hwc_to_chw(host(y).reshape(h, w, cout))
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-5 * max(np.abs(ref).max(), 1e-3))
    dx_ref, dw_ref, db_ref = oracle.conv_backward(g, x, wt, need_dx=True)
    dx_ref = dx_ref * (x > 0)
    need_dx = cin > 1
    d_dw, d_db = empty(wt.size), empty(cout)
    d_dx = empty(P * cin) if need_dx else None
    _call(lib, "n2f_conv_bwd", d_g.data_ptr(), d_x.data_ptr(), d_w.data_ptr(),
          d_x.data_ptr() if need_dx else None, d_dx.data_ptr() if need_dx else None,
          d_dw.data_ptr(), d_db.data_ptr(), h, w, cin, cout, k, IMPL, None)
    dw = engine_to_oihw(host(d_dw), cout, cin, k)
    np.testing.assert_allclose(dw, dw_ref, rtol=0, atol=1e-5 * max(np.abs(dw_ref).max(), 1e-3))
    np.testing.assert_allclose(host(d_db), db_ref, rtol=0, atol=1e-5 * max(np.abs(db_ref).max(), 1e-3))
    if need_dx:
        dx = hwc_to_chw(host(d_dx).reshape(h, w, cin))
        np.testing.assert_allclose(dx, dx_ref, rtol=0, atol=1e-5 * max(np.abs(dx_ref).max(), 1e-3))


@pytest.mark.parametrize("loss", [0, 1])
def test_loss(lib, oracle, loss):
    rng = np.random.default_rng(5 + loss)
    n = 70001
    z = (rng.standard_normal(n) * 6).astype(np.float32)
    z[:4] = [0.0, -40.0, 40.0, -0.0]
    t = rng.random(n).astype(np.float32)
    lv_ref, g_ref = (oracle.bce_logits if loss == 0 else oracle.mse_sigmoid)(z, t)
    g = empty(n)
    lv = C.c_double()
    d_z, d_t = dev(z), dev(t)
    _call(lib, "n2f_loss", d_z.data_ptr(), d_t.data_ptr(), g.data_ptr(), n, loss, C.byref(lv), None)
    # sigma(z) - t cancels when sigma(z) ~ t: bound the error by the grad scale
    np.testing.assert_allclose(host(g), g_ref, rtol=2e-6, atol=1e-6 * np.abs(g_ref).max())
    assert abs(lv.value - lv_ref) <= 1e-6 * abs(lv_ref)


def test_bce_known_answers(lib):
    z = np.array([0.0, -40.0, 40.0], np.float32)
    t = np.array([0.5, 0.0, 1.0], np.float32)
    g = empty(3)
    lv = C.c_double()
    d_z, d_t = dev(z), dev(t)
    _call(lib, "n2f_loss", d_z.data_ptr(), d_t.data_ptr(), g.data_ptr(), 3, 0, C.byref(lv), None)
    assert abs(lv.value - np.log(2) / 3) < 1e-7
    gg = host(g)
    assert gg[0] == 0.0 and abs(gg[1]) < 1e-12 and abs(gg[2]) < 1e-12


def test_adam_bitwise(lib, oracle, golden):
    p0 = golden["adam_p0"]
    grads = golden["adam_grads"]
    p, m, v = dev(p0), empty(p0.size), empty(p0.size)
    m.zero_()
    v.zero_()
    for k in range(grads.shape[0]):
        d_g = dev(grads[k])
        _call(lib, "n2f_adam", p.data_ptr(), d_g.data_ptr(), m.data_ptr(), v.data_ptr(),
              p0.size, k + 1, 0.003, None)
    assert np.array_equal(host(p), golden["adam_p"])
    assert np.array_equal(host(m), golden["adam_m"])
    assert np.array_equal(host(v), golden["adam_v"])


def test_adam_long_run_bitwise(lib, oracle):
    rng = np.random.default_rng(3)
    n = 4099
    p_ref = rng.standard_normal(n).astype(np.float32)
    m_ref, v_ref = np.zeros_like(p_ref), np.zeros_like(p_ref)
    p, m, v = dev(p_ref), empty(n), empty(n)
    m.zero_()
    v.zero_()
    for t in range(1, 301):
        g = (rng.standard_normal(n) * 10.0 ** rng.uniform(-9, 1, n)).astype(np.float32)
        oracle.adam_update(p_ref, g, m_ref, v_ref, t, 1e-3)
        d_g = dev(g)
        _call(lib, "n2f_adam", p.data_ptr(), d_g.data_ptr(), m.data_ptr(), v.data_ptr(), n, t,
              1e-3, None)
    assert np.array_equal(host(p), p_ref)
    assert np.array_equal(host(m), m_ref)
    assert np.array_equal(host(v), v_ref)


def test_validate_tail(lib, oracle):
    rng = np.random.default_rng(11)
    n = 50000
    z = (rng.standard_normal(n) * 5).astype(np.float32)
    z[:3] = [200.0, -200.0, 0.0]
    norm = rng.random(n).astype(np.float32)
    out_ref = np.clip(oracle.sigmoid(z), oracle.TINY32, oracle.TOP32)
    score_ref = oracle.val_score(out_ref, norm)
    out = empty(n)
    sc = C.c_double()
    d_z, d_n = dev(z), dev(norm)
    _call(lib, "n2f_validate_tail", d_z.data_ptr(), d_n.data_ptr(), out.data_ptr(), n,
          C.byref(sc), None)
    o = host(out)
    assert o.min() > 0 and o.max() < 1
    np.testing.assert_allclose(o, out_ref, rtol=2e-6, atol=0)
    assert abs(sc.value - score_ref) <= 1e-6 * score_ref


def _replay(lib, scores, patience):
    arr = np.asarray(scores, np.float64)
    out = C.c_int()
    _call(lib, "n2f_stop_replay", arr.ctypes.data, arr.size, patience, C.byref(out))
    return out.value


def test_stop_rule(lib, oracle):
    assert _replay(lib, [1.0, 0.9] + [0.95] * 100, 100) == 102
    assert _replay(lib, [1.0 / (e + 1) for e in range(300)], 100) == -1
    rng = np.random.default_rng(99)
    for _ in range(100):
        patience = int(rng.integers(1, 8))
        scores = rng.uniform(0, 1, int(rng.integers(1, 60))).round(2)
        tr = oracle.StopTracker(patience, 3)
        expect = -1
        for e, s in enumerate(scores):
            if tr.push(float(s), np.zeros(1)):
                expect = e + 1
                break
        assert _replay(lib, scores, patience) == expect


@pytest.mark.parametrize("n,window,first", [(1, 1, 0), (3, 5, 2), (100, 100, 37), (4, 4, 0)])
def test_window_mean_bitwise(lib, oracle, n, window, first):
    rng = np.random.default_rng(n + window)
    plane = 3001
    ring = (rng.random((window, plane)) * 0.98 + 0.01).astype(np.float32)
    order = [(first + k) % window for k in range(n)]
    ref = oracle.denormalize(oracle.window_mean([ring[s] for s in order]), -1.5, 7.25)
    out = empty(plane, np.float64)
    d_r = dev(ring)
    _call(lib, "n2f_window_mean", d_r.data_ptr(), window, first, n, plane, -1.5, 7.25,
          out.data_ptr(), None)
    assert np.array_equal(host(out), ref)


@pytest.mark.parametrize("cin,cout", [(64, 64), (256, 256)])
def test_conv_accuracy_vs_f64(lib, oracle, cin, cout):
    """Error of each conv implementation against an f64 evaluation of the same
    fp32 inputs (prints the numbers; bounds are the fp32-reassociation level)."""
    rng = np.random.default_rng(cin)
    h, w = 64, 96
    x = np.maximum(rng.standard_normal((cin, h, w)), 0).astype(np.float32)
    wt = (rng.standard_normal((cout, cin, 3, 3)) * np.sqrt(2.0 / (9 * cin))).astype(np.float32)
    b = np.zeros(cout, np.float32)
    exact = oracle.conv_forward(x.astype(np.float64), wt.astype(np.float64), b.astype(np.float64))
    blas = oracle.conv_forward(x, wt, b)
    scale = np.abs(exact).max()
    errs = {"oracle_fp32": np.abs(blas - exact).max() / scale}
    d_x, d_w, d_b = dev(chw_to_hwc(x)), dev(oihw_to_engine(wt)), dev(b)
    y = empty(h * w * cout)
    _call(lib, "n2f_conv_fwd", d_x.data_ptr(), d_w.data_ptr(), d_b.data_ptr(), y.data_ptr(),
          h, w, cin, cout, 3, 0, IMPL, None)
    got = hwc_to_chw(host(y).reshape(h, w, cout))
    errs["f16x3"] = np.abs(got - exact).max() / scale
    # signed bias: mean of (got - exact) * sign(exact), relative to mean |exact|
    errs["f16x3_bias"] = float(np.mean((got - exact) * np.sign(exact)) / np.mean(np.abs(exact)))
    print(f"cin={cin} cout={cout} max-err/scale: {errs}")
    assert errs["f16x3"] < 3e-5 and abs(errs["f16x3_bias"]) < 1e-5


@pytest.mark.parametrize("impl", [1, 2, 4])
def test_other_conv_impls_unsupported(lib, impl):
    """One implementation only (no multi-backend dispatch): any conv_impl other
    than 0 / 3 is N2F_ERR_UNSUPPORTED, for the per-kernel entry points and for
    a context."""
    from paper_2108_10209_b200 import TrainConfig, _lib

    d = empty(32 * 32 * 32)
    w = empty(32 * 9 * 32)
    b = empty(32)
    with pytest.raises(_lib.N2FError) as e:
        _call(lib, "n2f_conv_fwd", d.data_ptr(), w.data_ptr(), b.data_ptr(), d.data_ptr(), 32, 32,
              32, 32, 3, 1, impl, None)
    assert e.value.code == _lib.N2F_ERR_UNSUPPORTED
    cfg = _lib.N2FConfig()
    cfg.loss, cfg.scheme, cfg.lr = 0, 0, 1e-3
    cfg.patience_epochs, cfg.avg_window, cfg.max_epochs = 100, 100, 10
    cfg.conv_impl = impl
    h = C.c_void_p()
    with pytest.raises(_lib.N2FError) as e:
        _call(lib, "n2f_create", 0, 32, 32, C.byref(cfg), C.byref(h))
    assert e.value.code == _lib.N2F_ERR_UNSUPPORTED
    del TrainConfig
