"""The reference's own known-answer tests, run through the C-ABI kernels.

Each test restates one reference test (cited) on the device path: exact
integer-valued answers where the reference asserts equality, its tolerance
where it asserts closeness.
"""

import ctypes as C

import numpy as np
import pytest

from n2f_testutil import chw_to_hwc, dev, empty, hwc_to_chw, host, oihw_to_engine

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2108_10209_b200 import _lib

    return _lib


def _fwd(lib, x_chw, w_oihw, b, relu=0, impl=3):
    cin, h, w = x_chw.shape
    cout, k = w_oihw.shape[0], w_oihw.shape[-1]
    y = empty(h * w * cout)
    d_x, d_w, d_b = dev(chw_to_hwc(x_chw)), dev(oihw_to_engine(w_oihw)), dev(b)
    lib.call("n2f_conv_fwd", d_x.data_ptr(), d_w.data_ptr(), d_b.data_ptr(), y.data_ptr(), h, w, cin,
             cout, k, relu, impl, None)
    return hwc_to_chw(host(y).reshape(h, w, cout))


def test_forward_scalar_affine(lib):
    """test_tensor.py:55-66: 1x1 conv, w = 2, b = 1, x = 5 -> exactly 11."""
    out = _fwd(lib, np.full((1, 1, 1), 5.0, np.float32), np.full((1, 1, 1, 1), 2.0, np.float32),
               np.ones(1, np.float32))
    assert out.shape == (1, 1, 1) and out[0, 0, 0] == 11.0


def test_forward_box_sum_with_zero_padding(lib):
    """test_tensor.py:68-79: 3x3 box sum of ones with zero padding: centre 9,
    corners 4 (first-layer kernel, Cin = 1)."""
    out = _fwd(lib, np.ones((1, 3, 3), np.float32), np.ones((1, 1, 3, 3), np.float32),
               np.zeros(1, np.float32))[0]
    assert out[1, 1] == 9.0
    for corner in (out[0, 0], out[0, 2], out[2, 0], out[2, 2]):
        assert corner == 4.0
    for edge in (out[0, 1], out[1, 0], out[1, 2], out[2, 1]):
        assert edge == 6.0


@pytest.mark.parametrize("cin,cout", [(32, 32), (64, 128), (128, 256)])
@pytest.mark.parametrize("hw", [(3, 3), (40, 24), (17, 70)])
def test_forward_box_sum_tensor_cores(lib, cin, cout, hw):
    """The same known answer through the tcgen05 FP16x3 kernels (CTA-pair
    tiles, TMA zero-fill at every image border and tile edge): all-ones
    input and weights give exactly 9 / 6 / 4 x Cin (interior / edge / corner);
    every product and partial sum is a small integer, so the split-precision
    result must be exact."""
    out = _fwd(lib, np.ones((cin, *hw), np.float32), np.ones((cout, cin, 3, 3), np.float32),
               np.zeros(cout, np.float32))
    h, w = hw
    ny = np.full(h, 3.0)
    ny[0] -= 1
    ny[-1] -= 1
    nx = np.full(w, 3.0)
    nx[0] -= 1
    nx[-1] -= 1
    expect = (np.outer(ny, nx) * cin).astype(np.float32)
    assert np.array_equal(out, np.broadcast_to(expect, out.shape))


def test_backward_scalar_chain_rule(lib):
    """test_tensor.py:123-135: d/dx = w = 2, d/dw = x = 5, d/db = 1."""
    g = dev(np.ones(1, np.float32))
    x = dev(np.full(1, 5.0, np.float32))
    w = dev(np.full(1, 2.0, np.float32))
    dx, dw, db = empty(1), empty(1), empty(1)
    lib.call("n2f_conv_bwd", g.data_ptr(), x.data_ptr(), w.data_ptr(), None, dx.data_ptr(),
             dw.data_ptr(), db.data_ptr(), 1, 1, 1, 1, 1, 3, None)
    assert host(dx)[0] == 2.0 and host(dw)[0] == 5.0 and host(db)[0] == 1.0


def _adam(lib, p, g, m, v, t, lr=1e-3):
    lib.call("n2f_adam", p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), p.numel(), t, lr, None)


def test_adam_first_step_hand_value(lib):
    """test_tensor.py:313-319: p = 0, g = 1 -> p = -0.001 / (1 + 1e-8) (the
    engine runs the reference's fp32 path, so to fp32 rounding)."""
    p, g = dev(np.zeros(1, np.float32)), dev(np.ones(1, np.float32))
    m, v = dev(np.zeros(1, np.float32)), dev(np.zeros(1, np.float32))
    _adam(lib, p, g, m, v, 1)
    assert abs(float(host(p)[0]) - (-0.001 / (1.0 + 1e-8))) < 1e-10


def test_adam_zero_gradient_is_noop(lib):
    """test_tensor.py:322-328."""
    p0 = np.array([1.5, -2.0], np.float32)
    p, g = dev(p0), dev(np.zeros(2, np.float32))
    m, v = dev(np.zeros(2, np.float32)), dev(np.zeros(2, np.float32))
    _adam(lib, p, g, m, v, 1)
    assert np.array_equal(host(p), p0) and not host(m).any() and not host(v).any()


def test_adam_two_steps_match_script(lib):
    """test_tensor.py:331-338 (float64 script; fp32 engine -> fp32 tolerance)."""
    p0 = np.array([0.2, -0.4], np.float32)
    p, g = dev(p0), dev(np.ones(2, np.float32))
    m, v = dev(np.zeros(2, np.float32)), dev(np.zeros(2, np.float32))
    _adam(lib, p, g, m, v, 1)
    _adam(lib, p, g, m, v, 2)
    pp, mm, vv = p0.astype(np.float64), np.zeros(2), np.zeros(2)
    for t in (1, 2):
        mm = 0.9 * mm + 0.1
        vv = 0.999 * vv + 0.001
        pp = pp - 1e-3 * (mm / (1 - 0.9 ** t)) / (np.sqrt(vv / (1 - 0.999 ** t)) + 1e-8)
    assert np.max(np.abs(host(p) - pp)) < 1e-7


def test_checkerboard_worked_example(lib):
    """test_downsample.py:20-26 on the device gather: x = [[1,2,3,4],[5,6,7,8]]
    -> eu [[1,3],[6,8]], ou [[2,4],[5,7]], el [[1,6,3,8]], ol [[5,2,7,4]]
    (the engine gathers the normalised image, (x - 1) / 7)."""
    x = np.array([[1, 2, 3, 4], [5, 6, 7, 8]], np.float64)
    d_x = dev(x)
    plane = 2 * 2
    d_norm, d_in, d_tgt = empty(8), empty(4 * plane), empty(4 * plane)
    ph, pw = (C.c_int * 4)(), (C.c_int * 4)()
    lib.call("n2f_make_pairs", d_x.data_ptr(), lib.N2F_F64, None, 2, 4, 1.0, 8.0, 0, 0,
             d_norm.data_ptr(), d_in.data_ptr(), d_tgt.data_ptr(), ph, pw, None)
    nz = lambda a: ((np.asarray(a, np.float64) - 1.0) / 7.0).astype(np.float32)  # noqa: E731
    gin = host(d_in)
    expect = [[[1, 3], [6, 8]], [[2, 4], [5, 7]], [[1, 6, 3, 8]], [[5, 2, 7, 4]]]
    for k, e in enumerate(expect):
        e = np.array(e)
        assert (ph[k], pw[k]) == e.shape
        assert np.array_equal(gin[k * plane: k * plane + e.size].reshape(e.shape), nz(e))


def test_dead_relu_path_has_zero_weight_gradient(oracle):
    """test_model.py:175-186 through a full engine step: one first-layer unit
    driven permanently negative (bias -1e3) gets exactly zero weight and bias
    gradient; live units still learn."""
    from paper_2108_10209_b200 import Engine, TrainConfig, _lib
    from n2f_testutil import arena_to_layers, net_to_arena

    net = oracle.init_net(4)
    dead = 1
    net.biases[0][dead] = -1e3
    img = np.random.default_rng(10).uniform(0, 1, (32, 32))
    eng = Engine(32, 32, TrainConfig(seed=4), use_graph=False)
    _lib.call("n2f_ctx_prepare", eng.handle, img.ctypes.data, _lib.N2F_F64, None, 0)
    arena = net_to_arena(net)
    _lib.call("n2f_ctx_set_params", eng.handle, arena.ctypes.data)
    _lib.call("n2f_ctx_step", eng.handle, 0, None)
    n = C.c_int64()
    _lib.call("n2f_ctx_param_count", eng.handle, C.byref(n))
    grads = np.empty(n.value, np.float32)
    _lib.call("n2f_ctx_get_arena", eng.handle, 3, grads.ctypes.data)
    gw0, gb0 = arena_to_layers(grads, oracle.layer_shapes())[0]
    assert not gw0[dead].any() and gb0[dead] == 0.0
    assert gw0[0].any()
    eng.close()
