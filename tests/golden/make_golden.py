"""Generate the golden fixtures that pin ``oracle/n2f_oracle.py`` to the reference.

Run in the build container (the only place ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/nbc \
        python tests/golden/make_golden.py

It imports the real reference package read-only from
``/root/reference/pkg/src`` and calls its public functions on small seeded
inputs; the outputs are written to ``tests/golden/reference_vectors.npz``.
Large arrays (full-network weights) are stored as SHA-256 digests plus
per-layer norms and strided samples to keep the fixture small.
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.npz")


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def samples(a: np.ndarray, n: int = 64) -> np.ndarray:
    flat = np.ascontiguousarray(a).reshape(-1)
    idx = np.linspace(0, flat.size - 1, min(n, flat.size)).astype(np.int64)
    return flat[idx]


def main() -> None:
    sys.path.insert(0, REF)
    from noise2fast import downsample, imaging, model, rng, tensor, trainer  # noqa: E402

    g: dict[str, np.ndarray] = {}
    meta: dict = {}

    # --- rng (rng.py) ---------------------------------------------------
    seeds = [0, 1, 7, 123456789, 2**63 + 5]
    g["rng_derive"] = np.array(
        [rng.derive_seed(s, *ids) for s in seeds for ids in ((), (0,), (3,), (1, 2), (5, 0, 9))],
        dtype=np.uint64,
    )
    g["rng_uniform"] = np.concatenate([rng.CounterRng(s).uniform(97, -0.3, 0.7) for s in seeds])
    g["rng_normal"] = np.concatenate([rng.CounterRng(s).normal(33, 0.5) for s in seeds])

    # --- network init (model.py:46-65) ---------------------------------
    for s in (0, 7, 4242):
        net = model.build_network(1, s)
        for i, layer in enumerate(net.layers):
            g[f"init_s{s}_l{i}_samples"] = samples(layer.weights)
            meta[f"init_s{s}_l{i}_sha"] = digest(layer.weights)
    meta["param_count"] = int(model.parameter_count(model.build_network(1, 0)))

    # --- normalize / downsample ----------------------------------------
    r = np.random.default_rng(11)
    img = r.normal(3.0, 2.0, (13, 17))
    norm, p = imaging.normalize_plane(img)
    g["norm_in"], g["norm_out"] = img, norm
    g["norm_minmax"] = np.array([p.vmin, p.vmax])
    for hw in ((6, 8), (7, 9), (2, 2), (10, 4)):
        x = r.random(hw).astype(np.float32)
        g[f"ds_in_{hw[0]}x{hw[1]}"] = x
        for scheme in ("checkerboard", "quad"):
            pairs = downsample.make_training_pairs(x, scheme)
            for k, pr in enumerate(pairs):
                g[f"ds_{scheme}_{hw[0]}x{hw[1]}_{k}_in"] = pr.input
                g[f"ds_{scheme}_{hw[0]}x{hw[1]}_{k}_tgt"] = pr.target
        clean = r.random(hw).astype(np.float32)
        g[f"ds_clean_{hw[0]}x{hw[1]}"] = clean
        for k, pr in enumerate(downsample.make_exact_pairs(x, clean)):
            g[f"ds_exact_{hw[0]}x{hw[1]}_{k}_tgt"] = pr.target

    # --- conv fwd/bwd fp32 (tensor.py:490-530) --------------------------
    for j, (cin, cout, k, h, w) in enumerate(((1, 4, 3, 5, 7), (3, 5, 3, 6, 4), (4, 1, 1, 3, 5), (8, 8, 3, 9, 9))):
        x = r.standard_normal((1, cin, h, w)).astype(np.float32)
        wt = r.standard_normal((cout, cin, k, k)).astype(np.float32)
        b = r.standard_normal(cout).astype(np.float32)
        layer = tensor.ConvLayer(wt, b, (k - 1) // 2, "relu")
        out, pre = tensor.conv2d_forward(x, layer, return_preact=True)
        go = r.standard_normal(out.shape).astype(np.float32)
        gi, gw, gb = tensor.conv2d_backward(go, x, layer, preact=pre)
        for name, a in (("x", x), ("w", wt), ("b", b), ("pre", pre), ("go", go), ("gi", gi), ("gw", gw), ("gb", gb)):
            g[f"conv{j}_{name}"] = a

    # --- losses ----------------------------------------------------------
    z = (r.standard_normal((1, 1, 6, 7)) * 4).astype(np.float32)
    t = r.random((1, 1, 6, 7)).astype(np.float32)
    lv, gz = tensor.bce_with_logits(z, t)
    g["bce_z"], g["bce_t"], g["bce_grad"], g["bce_loss"] = z, t, gz, np.array([lv])
    s = tensor.sigmoid(z)
    mv, gs = tensor.mse_loss(s, t)
    g["mse_grad"], g["mse_loss"] = gs * s * (1 - s), np.array([mv])
    g["sigmoid_z"] = (r.standard_normal(200) * 30).astype(np.float32)
    g["sigmoid_out"] = tensor.sigmoid(g["sigmoid_z"])

    # --- Adam, 7 steps (tensor.py:125-141) ------------------------------
    prm = r.standard_normal(300).astype(np.float32)
    st = tensor.AdamState.zeros_like(prm, lr=0.003)
    g["adam_p0"] = prm.copy()
    grads = (r.standard_normal((7, 300)) * np.logspace(-9, 1, 300)).astype(np.float32)
    g["adam_grads"] = grads
    for k in range(7):
        tensor.adam_step(prm, grads[k], st)
    g["adam_p"], g["adam_m"], g["adam_v"] = prm, st.m, st.v

    # --- stop rule + finalize (trainer.py:78-109) -----------------------
    cfg = trainer.TrainConfig(patience_epochs=5, avg_window=4)
    seq = r.uniform(0, 1, 40).round(1)
    state = trainer.TrainState(avg_window=4)
    outs = (r.random((40, 3, 5)) * 0.9 + 0.05).astype(np.float32)
    stop = -1
    for e, sc in enumerate(seq):
        if trainer.update_stop_state(state, float(sc), outs[e], cfg) == "stop":
            stop = e + 1
            break
    g["stop_scores"], g["stop_outs"], g["stop_epoch"] = seq, outs, np.array([stop])
    g["stop_final"] = trainer.finalize_output(state, imaging.NormParams(-2.0, 5.0))

    # --- whole network: predict, 1 step, 1 epoch (model.py, trainer.py) -
    noisy = (r.random((16, 20)) * 3 - 1).astype(np.float64)
    norm, p = imaging.normalize_plane(noisy)
    n32 = norm.astype(np.float32)
    g["net_noisy"] = noisy
    net = model.build_network(1, 7)
    out0 = model.predict(net, n32)
    g["net_pred0"] = out0
    g["net_score0"] = np.array([trainer.validate(net, n32)[0]])
    pairs = downsample.make_training_pairs(n32, "checkerboard")
    for k, pr in enumerate(pairs):
        logits, cache = model.forward(net, pr.input[None, None], keep_cache=True)
        lv, gz = tensor.bce_with_logits(logits, np.clip(pr.target, 0, 1)[None, None])
        grads = model.backward(net, cache, gz)
        if k == 0:
            g["net_step1_logits"] = logits[0, 0]
            g["net_step1_loss"] = np.array([lv])
            for i, (gw, gb) in enumerate(grads):
                g[f"net_step1_gw{i}_samples"] = samples(gw)
                g[f"net_step1_gb{i}"] = gb
                meta[f"net_step1_gw{i}_sha"] = digest(gw)
                g[f"net_step1_gw{i}_norm"] = np.array([np.linalg.norm(gw.astype(np.float64))])
        model.apply_gradients(net, grads)
        if k == 0:
            for i, layer in enumerate(net.layers):
                meta[f"net_step1_w{i}_sha"] = digest(layer.weights)
                g[f"net_step1_w{i}_samples"] = samples(layer.weights)
    for i, layer in enumerate(net.layers):
        meta[f"net_epoch1_w{i}_sha"] = digest(layer.weights)
        g[f"net_epoch1_w{i}_samples"] = samples(layer.weights)
        g[f"net_epoch1_b{i}"] = layer.bias
    g["net_epoch1_pred"] = model.predict(net, n32)

    # --- a short full run (trainer.py:125-213) ---------------------------
    cfg = trainer.TrainConfig(seed=3, patience_epochs=2, avg_window=3, max_epochs=5)
    buf = io.StringIO()
    res = trainer.train_single_channel(noisy[:12, :14], cfg, telemetry=buf)
    g["run_denoised"] = res.denoised
    g["run_history"] = np.array(res.val_history)
    meta["run_epochs"] = res.epochs_run
    meta["run_reason"] = res.stop_reason
    meta["run_losses"] = [json.loads(line)["train_loss_per_pair"] for line in buf.getvalue().splitlines()]
    for loss, scheme in (("mse", "checkerboard"), ("bce", "quad")):
        cfg = trainer.TrainConfig(seed=5, patience_epochs=2, avg_window=2, max_epochs=3, loss=loss, scheme=scheme)
        res = trainer.train_single_channel(noisy[:10, :12], cfg)
        g[f"run_{loss}_{scheme}_denoised"] = res.denoised
        g[f"run_{loss}_{scheme}_history"] = np.array(res.val_history)

    g["meta_json"] = np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
