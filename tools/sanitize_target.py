"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): a 64^2 fit of 2 epochs with every kernel launched from the host
(tcgen05 conv/dgrad/wgrad CTA pairs, first-layer kernels, fused heads, Adam,
stop rule, window mean), then one CUDA-graph fit of the same image.

    compute-sanitizer --tool racecheck python tools/sanitize_target.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2108_10209_b200 import Engine, TrainConfig, synthetic  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 64
clean = synthetic.blob_rect_image(size, size, 3)
noisy = synthetic.gaussian_noisy(clean, 25 / 255, 4).astype(np.float64)
cfg = TrainConfig(seed=1, max_epochs=2, patience_epochs=100, avg_window=2)
for graph in (False, True):
    eng = Engine(size, size, cfg, use_graph=graph)
    out, r, hist, _, _ = eng.fit_host(np.ascontiguousarray(noisy))
    eng.close()
    print(f"graph={graph} epochs={r.epochs_run} launches={r.kernel_launches} val={hist.tolist()} "
          f"finite={bool(np.isfinite(out).all())}")
