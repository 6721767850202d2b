"""ncu workload for the HBM-bound per-fit kernels at the config-5 size
(4096^2): one 1-epoch fit (min/max scan, normalise, pair gather, init,
window mean), host-loop mode so every kernel is a separate launch."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2108_10209_b200 import Engine, TrainConfig, synthetic  # noqa: E402

noisy, _ = synthetic.config_image(5, 0)
eng = Engine(4096, 4096, TrainConfig(seed=0, max_epochs=1, avg_window=1), use_graph=False)
out, r, hist, _, _ = eng.fit_host(np.ascontiguousarray(noisy))
print("epochs", r.epochs_run, "val", hist.tolist())
