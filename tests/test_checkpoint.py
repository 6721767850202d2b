"""N2FW weight checkpoints (model.py:143-184) from / into the engine arena.

CPU: the seeded networks written from the engine-layout arena are
byte-identical to the reference's own checkpoints (SHA-256 digests generated
by importing the reference, tests/golden/make_golden_checkpoint.py), round
trip exactly, and bad files raise the reference's errors.  GPU: a fitted
context's checkpoint, loaded into the CPU oracle, predicts what the context
validates.
"""

import hashlib
import json
import os
import struct

import numpy as np
import pytest

from n2f_testutil import net_to_arena, norm_rel

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "checkpoint_digests.json")


@pytest.mark.parametrize("seed", [0, 7, 4242])
def test_checkpoint_bytes_match_reference(oracle, tmp_path, seed):
    from paper_2108_10209_b200 import checkpoint

    want = json.load(open(GOLDEN))[str(seed)]
    path = tmp_path / "w.n2fw"
    arena = net_to_arena(oracle.init_net(seed))
    checkpoint.save_checkpoint(arena, path, seed)
    data = path.read_bytes()
    assert len(data) == want["bytes"]
    assert hashlib.sha256(data).hexdigest() == want["sha256"]
    back, s, cin = checkpoint.load_checkpoint(path)
    assert s == seed and cin == 1 and np.array_equal(back, arena)


def test_checkpoint_errors(tmp_path):
    """test_model.py:249-262: bad magic / unsupported version."""
    from paper_2108_10209_b200 import checkpoint

    bad = tmp_path / "bad.n2fw"
    bad.write_bytes(b"XXXX" + b"\0" * 64)
    with pytest.raises(ValueError, match="bad magic"):
        checkpoint.load_checkpoint(bad)
    v2 = tmp_path / "v2.n2fw"
    v2.write_bytes(b"N2FW" + struct.pack("<III", 2, 1, 9) + b"\0" * 64)
    with pytest.raises(ValueError, match="unsupported checkpoint version 2"):
        checkpoint.load_checkpoint(v2)


@pytest.mark.gpu
def test_fitted_checkpoint_predicts_like_the_context(oracle, tmp_path):
    import ctypes as C

    from paper_2108_10209_b200 import Engine, TrainConfig, _lib, checkpoint, synthetic

    clean = synthetic.blob_rect_image(64, 48, 5)
    img = synthetic.gaussian_noisy(clean, 25 / 255, 6).astype(np.float64)
    eng = Engine(64, 48, TrainConfig(seed=3, max_epochs=3), use_graph=False)
    eng.fit_host(np.ascontiguousarray(img))
    path = tmp_path / "fit.n2fw"
    eng.save_checkpoint(path)
    out = np.empty(img.size, np.float32)
    score = C.c_double()
    _lib.call("n2f_ctx_validate", eng.handle, out.ctypes.data, C.byref(score))
    arena, seed, _ = checkpoint.load_checkpoint(path)
    assert seed == 3 and np.array_equal(arena, eng.params())
    net = oracle.init_net(0)
    for i, (w, b) in enumerate(checkpoint.arena_to_layers(arena)):
        net.weights[i], net.biases[i] = w.copy(), b.copy()
    n32 = oracle.normalize(img)[0].astype(np.float32)
    assert norm_rel(out.reshape(img.shape), oracle.predict(net, n32)) < 1e-4
    # and back: loading the checkpoint into a fresh context reproduces the output
    eng2 = Engine(64, 48, TrainConfig(seed=3), use_graph=False)
    _lib.call("n2f_ctx_prepare", eng2.handle, img.ctypes.data, _lib.N2F_F64, None, 1)
    eng2.load_checkpoint(path)
    out2 = np.empty(img.size, np.float32)
    _lib.call("n2f_ctx_validate", eng2.handle, out2.ctypes.data, C.byref(score))
    assert np.array_equal(out, out2)
    eng.close()
    eng2.close()
