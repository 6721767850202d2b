"""Small, deterministic GPU workload for ncu: one bounded fit (2 epochs) of the
bench image (512x512, config 2) through the engine in host-loop mode, so
every kernel is a separate, attributable launch."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2108_10209_b200 import Engine, TrainConfig, synthetic  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 2
noisy, _ = synthetic.config_image(2, 0)
eng = Engine(512, 512, TrainConfig(seed=0, max_epochs=epochs, patience_epochs=10**6), use_graph=False)
out, r, hist, _, _ = eng.fit_host(np.ascontiguousarray(noisy))
print(f"epochs {r.epochs_run} gpu_ms {r.gpu_ms:.1f} launches {r.kernel_launches} val {hist.tolist()}")
