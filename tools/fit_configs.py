"""Full default fits of the BASELINE.json configs 3 (1024^2 microscopy) and
5 (4096^2 blob+rectangle) through the public API: epochs, device time,
ms/epoch, PSNR against the known clean image.  One JSON line per config.

    python tools/fit_configs.py [--configs 3 5]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2108_10209_b200 import Engine, TrainConfig, synthetic  # noqa: E402


def psnr(a, b):
    return float(10 * np.log10(1.0 / np.mean((np.asarray(a, np.float64) - b) ** 2)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[3, 5])
    args = ap.parse_args()
    for cfgn in args.configs:
        noisy, clean = synthetic.config_image(cfgn, 0)
        h, w = noisy.shape
        eng = Engine(h, w, TrainConfig(seed=0))
        t0 = time.perf_counter()
        out, r, hist, _, _ = eng.fit_host(np.ascontiguousarray(noisy))
        wall = time.perf_counter() - t0
        print(json.dumps({
            "config": cfgn, "image": [h, w], "epochs_run": int(r.epochs_run),
            "stop_reason": int(r.stop_reason), "gpu_ms": r.gpu_ms, "wall_s": wall,
            "ms_per_epoch": r.gpu_ms / max(1, r.epochs_run), "images_per_s": 1.0 / wall,
            "context_gib": eng.device_bytes / 2**30,
            "psnr_noisy_db": psnr(noisy, clean),  # both on the noisy image's [0, 1] scale
            "psnr_denoised_db": psnr(out, clean)}), flush=True)
        eng.close()


if __name__ == "__main__":
    main()
