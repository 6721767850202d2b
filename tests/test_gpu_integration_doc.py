"""The reference-side ctypes binding printed in INTEGRATION.md is executed as
written (only the library path is made absolute) and must reproduce
train_single_channel bit for bit: the documented drop-in recipe cannot rot."""

import os
import re
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _binding_source():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    src = next(b for b in blocks if "noise2fast/_b200.py" in b)
    lib = os.path.join(ROOT, "paper_2108_10209_b200", "libn2f.so")
    assert 'ctypes.CDLL("libn2f.so")' in src
    return src.replace('ctypes.CDLL("libn2f.so")', f"ctypes.CDLL({lib!r})")


def test_documented_binding_matches_public_api():
    from paper_2108_10209_b200 import TrainConfig, synthetic, train_single_channel

    mod = types.ModuleType("n2f_doc_binding")
    exec(compile(_binding_source(), "INTEGRATION.md", "exec"), mod.__dict__)
    clean = synthetic.blob_rect_image(48, 40, 5)
    noisy = synthetic.gaussian_noisy(clean, 25 / 255, 6).astype(np.float64)
    cfg = TrainConfig(seed=9, patience_epochs=4, avg_window=3, max_epochs=6)
    out = mod.fit(noisy, cfg)
    ref = train_single_channel(noisy, cfg)
    assert out.dtype == np.float64 and out.shape == noisy.shape
    assert np.array_equal(out, ref.denoised)
    bad = noisy.copy()
    bad[3, 4] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        mod.fit(bad, cfg)
