"""Out-of-bounds write check on the whole engine (compute-sanitizer is not
available on the GPU pool): every context allocation is bracketed by guard
bytes (engine.cu dalloc); after fits at ragged, minimum and BASELINE sizes,
every scheme / loss, host-loop and graph, no guard may have changed."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _guards(eng):
    from paper_2108_10209_b200 import _lib

    n = C.c_int(-1)
    _lib.call("n2f_ctx_check_guards", eng.handle, C.byref(n))
    return n.value


@pytest.mark.parametrize("hw", [(4, 4), (5, 7), (16, 9), (33, 47), (130, 66), (64, 64), (257, 511), (4, 1030),
                                (1030, 4)])
@pytest.mark.parametrize("scheme,loss", [("checkerboard", "bce"), ("quad", "mse"), ("exact", "bce")])
@pytest.mark.parametrize("use_graph", [False, True])
def test_no_out_of_bounds_writes(hw, scheme, loss, use_graph):
    from paper_2108_10209_b200 import Engine, TrainConfig

    rng = np.random.default_rng(hash((hw, scheme)) % 2**32)
    img = rng.random(hw)
    clean = rng.random(hw) if scheme == "exact" else None
    eng = Engine(*hw, TrainConfig(seed=3, scheme=scheme, loss=loss, max_epochs=3, patience_epochs=2,
                                  avg_window=2), use_graph=use_graph)
    assert _guards(eng) == 0
    out, r, _, _, _ = eng.fit_host(np.ascontiguousarray(img), clean)
    assert r.epochs_run >= 1 and np.isfinite(out).all()
    assert _guards(eng) == 0
    eng.close()


def test_no_out_of_bounds_writes_config2_epochs():
    from paper_2108_10209_b200 import Engine, TrainConfig, synthetic

    noisy, _ = synthetic.config_image(2, 0)
    eng = Engine(512, 512, TrainConfig(seed=0, max_epochs=4, patience_epochs=100))
    eng.fit_host(np.ascontiguousarray(noisy))
    assert _guards(eng) == 0
    eng.close()
