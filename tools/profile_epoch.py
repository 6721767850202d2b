"""Per-kernel-class / per-layer timing of one training epoch at a given size
(CUDA events around every launch), with achieved algorithmic TFLOP/s.

    python tools/profile_epoch.py --size 512
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2108_10209_b200 import Engine, TrainConfig, synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    clean = synthetic.blob_rect_image(args.size, args.size, 0)
    noisy = synthetic.gaussian_noisy(clean, 50 / 255, 1)
    eng = Engine(args.size, args.size, TrainConfig(seed=0, max_epochs=3, patience_epochs=10**6))
    eng.fit_host(np.ascontiguousarray(noisy))  # warm up + leaves a prepared context
    print(f"context device bytes: {eng.device_bytes / 2**30:.2f} GiB")
    ms, fl, ln = eng.profile_epoch()
    total = ms.sum()
    rows = []
    for ci, name in enumerate(Engine.PROF_CLASSES):
        for li in range(9):
            if ln[ci, li] == 0:
                continue
            t = float(ms[ci, li])
            tf = float(fl[ci, li]) / (t * 1e-3) / 1e12 if fl[ci, li] > 0 else None
            rows.append({"class": name, "layer": li + 1, "launches": int(ln[ci, li]), "ms": round(t, 4),
                         "ms_per_launch": round(t / ln[ci, li], 4), "share": round(t / total, 4),
                         "tflops": None if tf is None else round(tf, 1)})
    for r in sorted(rows, key=lambda r: -r["ms"]):
        print(f"{r['class']:12s} L{r['layer']}  n={r['launches']:2d}  {r['ms']:8.3f} ms  "
              f"{100 * r['share']:5.1f}%  {r['tflops'] if r['tflops'] is not None else '':>7} TF/s")
    print(f"epoch total {total:.3f} ms")
    if args.json:
        with open(args.json, "w") as f:
            json.dump({"size": args.size, "epoch_ms": total, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
