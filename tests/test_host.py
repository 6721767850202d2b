"""CPU-only checks: the C-ABI library loads and exports every symbol declared
in include/n2f.h, and the host-side mirror of the reference API behaves like
the reference before any device work (config validation, argument errors,
seed derivation)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "n2f.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(n2f_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2108_10209_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes signature table covers the same set
    assert set(_lib.SIGNATURES) == set(syms)


def test_library_loads_without_gpu():
    from paper_2108_10209_b200 import _lib

    lib = _lib.load()
    assert lib.n2f_version().startswith(b"n2f-b200")


def test_library_is_sm100a():
    import subprocess

    from paper_2108_10209_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_trainconfig_validation_matches_reference():
    from paper_2108_10209_b200 import TrainConfig

    TrainConfig()
    for kw, msg in [({"loss": "l1"}, "loss must be one of"), ({"scheme": "x"}, "scheme must be one of"),
                    ({"lr": 0}, "lr must be > 0"), ({"patience_epochs": 0}, "patience_epochs"),
                    ({"avg_window": 0}, "avg_window"), ({"max_epochs": 0}, "max_epochs")]:
        with pytest.raises(ValueError, match=msg):
            TrainConfig(**kw)


def test_argument_errors_raise_before_device_work():
    from paper_2108_10209_b200 import TrainConfig, train_single_channel

    cfg = TrainConfig()
    with pytest.raises(ValueError, match="expected a 2-D image"):
        train_single_channel(np.zeros((5, 5, 2)), cfg)
    with pytest.raises(ValueError, match="at least 4x4"):
        train_single_channel(np.zeros((3, 9)), cfg)
    with pytest.raises(ValueError, match="exact scheme requires"):
        train_single_channel(np.ones((6, 6)), TrainConfig(scheme="exact"))
    with pytest.raises(ValueError, match="clean shape"):
        train_single_channel(np.ones((6, 6)), TrainConfig(scheme="exact"), clean=np.ones((6, 7)))
    with pytest.raises(ValueError, match="non-finite"):
        train_single_channel(np.full((6, 6), np.nan), TrainConfig(scheme="exact"), clean=np.ones((6, 6)))


def test_derive_seed_matches_oracle(oracle):
    from paper_2108_10209_b200 import derive_seed

    for s in (0, 1, 7, 2**63 + 11, 2**64 - 1):
        for ids in ((), (0,), (2, 3), (1, 0, 5)):
            assert derive_seed(s, *ids) == oracle.child_seed(s, *ids)


def test_denoise_image_channel_checks():
    from paper_2108_10209_b200 import ImageData, TrainConfig, denoise_image

    img = ImageData(np.zeros((1, 8, 8, 5), np.float32))
    with pytest.raises(ValueError, match="1-4 channels"):
        denoise_image(img, TrainConfig())


def test_device_selection_for_pool_workers():
    """N2F_DEVICE=auto maps pool worker i to GPU i mod count (one image per GPU
    at a time under the reference CLI's --threads pool, cli.py:207-211)."""
    from paper_2108_10209_b200.trainer import select_device

    assert select_device(None, 5, 8) == 0
    assert select_device("3", 5, 8) == 3
    assert [select_device("auto", i, 4) for i in range(9)] == [0, 1, 2, 3, 0, 1, 2, 3, 0]
    with pytest.raises(RuntimeError, match="no CUDA device"):
        select_device("auto", 0, 0)


def test_metrics_argument_errors_before_device_work():
    """Reference error behaviour of imaging.psnr / imaging.ssim (imaging.py:255-300)."""
    from paper_2108_10209_b200 import metrics

    with pytest.raises(ValueError, match="shape mismatch"):
        metrics.psnr(np.zeros((2, 2)), np.zeros((2, 3)), 255.0)
    with pytest.raises(ValueError, match="data_range must be positive"):
        metrics.psnr(np.zeros((2, 2)), np.zeros((2, 2)), 0.0)
    with pytest.raises(ValueError, match="smaller than the 11x11 window"):
        metrics.ssim(np.zeros((10, 12)), np.zeros((10, 12)), 1.0)
    with pytest.raises(ValueError, match="single-channel 2-D"):
        metrics.ssim(np.zeros((12, 12, 3)), np.zeros((12, 12, 3)), 1.0)
    with pytest.raises(ValueError, match="shape mismatch"):
        metrics.ssim(np.zeros((12, 12)), np.zeros((12, 13)), 1.0)


def _hold_device_lock(i, q):
    import time

    from paper_2108_10209_b200.trainer import _device_lock

    with _device_lock(0):
        t0 = time.time()
        time.sleep(0.25)
        q.put((i, t0, time.time()))


def test_device_lock_serialises_processes_sharing_a_gpu():
    """Processes that share a GPU (CLI --threads N with fewer GPUs than
    workers) take turns per fit: the per-device file lock of the public API."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_hold_device_lock, args=(i, q)) for i in range(3)]
    for p in ps:
        p.start()
    iv = sorted((q.get(timeout=60) for _ in ps), key=lambda x: x[1])
    for p in ps:
        p.join(30)
    for (_, _, end), (_, start, _) in zip(iv, iv[1:]):
        assert end <= start + 1e-3, iv
