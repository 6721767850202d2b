"""Pin the CPU oracle (oracle/n2f_oracle.py) to the reference's own outputs.

The fixtures in tests/golden/reference_vectors.npz were produced by importing
the real reference package (tests/golden/make_golden.py).  Bit-exact where
the reference arithmetic is order-determined; the BLAS-backed convolutions
are compared at fp32 reassociation tolerance (the reference's own bar,
test_tensor.py:82-88 uses 1e-5 of array scale).
"""

import hashlib

import numpy as np
import pytest


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_rng_streams_bitwise(golden, oracle):
    seeds = [0, 1, 7, 123456789, 2**63 + 5]
    got = [oracle.child_seed(s, *ids) for s in seeds for ids in ((), (0,), (3,), (1, 2), (5, 0, 9))]
    assert np.array_equal(np.array(got, dtype=np.uint64), golden["rng_derive"])
    u = np.concatenate([oracle.counter_uniform(s, 97, -0.3, 0.7) for s in seeds])
    assert np.array_equal(u, golden["rng_uniform"])
    nrm = np.concatenate([oracle.counter_normal(s, 33, 0.5) for s in seeds])
    np.testing.assert_allclose(nrm, golden["rng_normal"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("seed", [0, 7, 4242])
def test_init_bitwise(golden, oracle, seed):
    net = oracle.init_net(seed)
    for i, w in enumerate(net.weights):
        assert sha(w) == golden["meta"][f"init_s{seed}_l{i}_sha"], i


def test_param_count(golden, oracle):
    net = oracle.init_net(0)
    n = sum(w.size + b.size for w, b in zip(net.weights, net.biases))
    assert n == golden["meta"]["param_count"] == 1171937


def test_normalize_bitwise(golden, oracle):
    norm, lo, hi, degen = oracle.normalize(golden["norm_in"])
    assert not degen
    assert np.array_equal(norm, golden["norm_out"])
    assert [lo, hi] == golden["norm_minmax"].tolist()


@pytest.mark.parametrize("hw", [(6, 8), (7, 9), (2, 2), (10, 4)])
@pytest.mark.parametrize("scheme", ["checkerboard", "quad", "exact"])
def test_pairs_bitwise(golden, oracle, hw, scheme):
    tag = f"{hw[0]}x{hw[1]}"
    x = golden[f"ds_in_{tag}"]
    clean = golden[f"ds_clean_{tag}"]
    pairs = oracle.training_pairs(x, scheme, clean)
    for k, (a, b) in enumerate(pairs):
        if scheme == "exact":
            assert np.array_equal(b, golden[f"ds_exact_{tag}_{k}_tgt"])
        else:
            assert np.array_equal(a, golden[f"ds_{scheme}_{tag}_{k}_in"])
            assert np.array_equal(b, golden[f"ds_{scheme}_{tag}_{k}_tgt"])


def test_checkerboard_worked_example(oracle):
    # 2x4 worked example (same numbers as test_downsample.py:20-26)
    x = np.arange(8).reshape(2, 4)
    eu, ou, el, ol = oracle.checkerboard(x)
    assert eu.tolist() == [[0, 2], [5, 7]]
    assert ou.tolist() == [[1, 3], [4, 6]]
    assert el.tolist() == [[0, 5, 2, 7]]
    assert ol.tolist() == [[4, 1, 6, 3]]


@pytest.mark.parametrize("j", range(4))
def test_conv_fwd_bwd(golden, oracle, j):
    x, w, b = golden[f"conv{j}_x"][0], golden[f"conv{j}_w"], golden[f"conv{j}_b"]
    pre = oracle.conv_forward(x, w, b)
    scale = np.abs(golden[f"conv{j}_pre"]).max()
    np.testing.assert_allclose(pre, golden[f"conv{j}_pre"][0], atol=1e-5 * scale, rtol=0)
    gp = golden[f"conv{j}_go"][0] * (pre > 0)
    gi, gw, gb = oracle.conv_backward(gp, x, w, need_dx=True)
    for name, got in (("gi", gi), ("gw", gw), ("gb", gb)):
        ref = golden[f"conv{j}_{name}"]
        ref = ref[0] if name == "gi" else ref
        np.testing.assert_allclose(got, ref, atol=1e-5 * np.abs(ref).max(), rtol=0)


def test_losses(golden, oracle):
    z, t = golden["bce_z"], golden["bce_t"]
    lv, gz = oracle.bce_logits(z, t)
    assert np.array_equal(gz, golden["bce_grad"])
    assert lv == golden["bce_loss"][0]
    lv, gm = oracle.mse_sigmoid(z, t)
    assert np.array_equal(gm, golden["mse_grad"])
    assert lv == golden["mse_loss"][0]
    assert np.array_equal(oracle.sigmoid(golden["sigmoid_z"]), golden["sigmoid_out"])


def test_bce_known_answers(oracle):
    lv, g = oracle.bce_logits(np.zeros((1, 1), np.float32), np.full((1, 1), 0.5, np.float32))
    assert abs(lv - np.log(2)) < 1e-6 and g[0, 0] == 0
    lv, g = oracle.bce_logits(np.array([[-40.0, 40.0]], np.float32), np.array([[0.0, 1.0]], np.float32))
    assert lv < 1e-12 and np.all(np.abs(g) < 1e-12)


def test_adam_bitwise(golden, oracle):
    p = golden["adam_p0"].copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    for k in range(7):
        oracle.adam_update(p, golden["adam_grads"][k], m, v, k + 1, 0.003)
    assert np.array_equal(p, golden["adam_p"])
    assert np.array_equal(m, golden["adam_m"])
    assert np.array_equal(v, golden["adam_v"])


def test_adam_first_step_known_answer(oracle):
    p = np.zeros(1, np.float32)
    m, v = np.zeros_like(p), np.zeros_like(p)
    oracle.adam_update(p, np.ones(1, np.float32), m, v, 1, 0.001)
    assert abs(p[0] - (-0.001 / (1 + 1e-8))) < 1e-9


def test_stop_and_window(golden, oracle):
    tr = oracle.StopTracker(5, 4)
    stop = -1
    for e, s in enumerate(golden["stop_scores"]):
        if tr.push(float(s), golden["stop_outs"][e]):
            stop = e + 1
            break
    assert stop == golden["stop_epoch"][0]
    out = oracle.denormalize(oracle.window_mean(tr.ring), -2.0, 5.0)
    assert np.array_equal(out, golden["stop_final"])


def test_stop_worked_schedule(oracle):
    tr = oracle.StopTracker(100, 100)
    z = np.zeros((1, 1), np.float32)
    stops = [tr.push(s, z) for s in [1.0, 0.9] + [0.95] * 100]
    assert stops.index(True) + 1 == 102


def test_network_predict_step_epoch(golden, oracle):
    noisy = golden["net_noisy"]
    norm, lo, hi, _ = oracle.normalize(noisy)
    n32 = norm.astype(np.float32)
    net = oracle.init_net(7)
    out0 = oracle.predict(net, n32)
    np.testing.assert_allclose(out0, golden["net_pred0"], rtol=0, atol=1e-6)
    pairs = oracle.training_pairs(n32)
    for k, (a, b) in enumerate(pairs):
        z, cache = oracle.net_forward(net, a, keep=True)
        lv, gz = oracle.bce_logits(z, b)
        grads = oracle.net_backward(net, cache, gz)
        if k == 0:
            np.testing.assert_allclose(z, golden["net_step1_logits"], rtol=0, atol=1e-6)
            for i, (gw, gb) in enumerate(grads):
                # same GEMM shapes as the reference -> bitwise equal on the same BLAS
                assert sha(gw) == golden["meta"][f"net_step1_gw{i}_sha"], i
        oracle.net_step(net, grads, 1e-3)
        if k == 0:
            for i, w in enumerate(net.weights):
                assert sha(w) == golden["meta"][f"net_step1_w{i}_sha"], i
                np.testing.assert_allclose(
                    w.reshape(-1)[np.linspace(0, w.size - 1, min(64, w.size)).astype(np.int64)],
                    golden[f"net_step1_w{i}_samples"], rtol=0, atol=1e-6)
    for i, w in enumerate(net.weights):
        assert sha(w) == golden["meta"][f"net_epoch1_w{i}_sha"], i
        ref = golden[f"net_epoch1_w{i}_samples"]
        got = w.reshape(-1)[np.linspace(0, w.size - 1, min(64, w.size)).astype(np.int64)]
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-5)
    np.testing.assert_allclose(oracle.predict(net, n32), golden["net_epoch1_pred"], rtol=0, atol=1e-5)


def test_short_full_run(golden, oracle):
    noisy = golden["net_noisy"][:12, :14]
    res = oracle.fit_denoise(noisy, seed=3, patience=2, window=3, max_epochs=5)
    assert res.epochs_run == golden["meta"]["run_epochs"]
    assert res.stop_reason == golden["meta"]["run_reason"]
    np.testing.assert_allclose(res.val_history, golden["run_history"], rtol=1e-6)
    np.testing.assert_allclose(res.denoised, golden["run_denoised"], rtol=0, atol=1e-5)
    np.testing.assert_allclose(res.train_losses, golden["meta"]["run_losses"], rtol=1e-5)


@pytest.mark.parametrize("loss,scheme", [("mse", "checkerboard"), ("bce", "quad")])
def test_variant_runs(golden, oracle, loss, scheme):
    noisy = golden["net_noisy"][:10, :12]
    res = oracle.fit_denoise(noisy, seed=5, patience=2, window=2, max_epochs=3, loss=loss, scheme=scheme)
    np.testing.assert_allclose(res.val_history, golden[f"run_{loss}_{scheme}_history"], rtol=1e-6)
    np.testing.assert_allclose(res.denoised, golden[f"run_{loss}_{scheme}_denoised"], rtol=0, atol=1e-5)


def test_degenerate(oracle):
    res = oracle.fit_denoise(np.full((6, 6), 3.5))
    assert res.stop_reason == "degenerate" and res.epochs_run == 0
    assert np.array_equal(res.denoised, np.full((6, 6), 3.5))


def test_metrics_oracle_matches_reference():
    """oracle.psnr / oracle.ssim vs the reference's own values
    (tests/golden/make_golden_metrics.py)."""
    import os

    import numpy as np

    from oracle import n2f_oracle as o

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "metrics_vectors.npz"))
    for k in range(int(z["ncases"])):
        a, b, r = z[f"a{k}"], z[f"b{k}"], float(z[f"range{k}"])
        assert abs(o.psnr(a, b, r) - float(z[f"psnr{k}"])) <= 1e-12 * abs(float(z[f"psnr{k}"]))
        assert abs(o.ssim(a, b, r) - float(z[f"ssim{k}"])) <= 1e-12
