"""Steady-state ms per epoch of the captured CUDA graph (the bench's code
path): a fixed-length fit (max_epochs = N, no early stop) timed on the device,
minus a 1-epoch fit to remove the fixed per-fit work.

    python tools/graph_epoch.py [--size 512] [--epochs 60]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2108_10209_b200 import Engine, TrainConfig, synthetic  # noqa: E402


def fit_ms(size, epochs, img):
    eng = Engine(size, size, TrainConfig(seed=0, max_epochs=epochs, patience_epochs=10**6))
    eng.fit_host(img)  # warm-up (graph instantiation, first-touch)
    best = float("inf")
    for _ in range(3):
        _, r, _, _, _ = eng.fit_host(img)
        best = min(best, r.gpu_ms)
    eng.close()
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--epochs", type=int, default=60)
    args = ap.parse_args()
    clean = synthetic.blob_rect_image(args.size, args.size, 0)
    img = np.ascontiguousarray(synthetic.gaussian_noisy(clean, 50 / 255, 1))
    t1 = fit_ms(args.size, 1, img)
    tn = fit_ms(args.size, args.epochs, img)
    print(f"graph: {args.epochs} epochs {tn:.2f} ms, 1 epoch {t1:.2f} ms -> "
          f"{(tn - t1) / (args.epochs - 1):.3f} ms/epoch steady state")


if __name__ == "__main__":
    main()
