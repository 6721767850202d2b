"""Full-fit PSNR parity across seeds: CPU oracle vs the GPU engine (SIMT,
tcgen05 3xTF32 and FP16x3 convs).  Prints one JSON line per (seed) and a summary.

    python tools/psnr_parity.py --size 64 --seeds 4
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import n2f_oracle as o  # noqa: E402
from paper_2108_10209_b200 import Engine, TrainConfig, synthetic  # noqa: E402


def psnr(a, b):
    return 10 * np.log10(1.0 / np.mean((np.asarray(a, np.float64) - b) ** 2))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=64)
    ap.add_argument("--seeds", type=int, default=4)
    ap.add_argument("--sigma", type=float, default=25.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-only", action="store_true")
    ap.add_argument("--first-seed", type=int, default=0)
    args = ap.parse_args()
    rows = []
    for s in range(args.first_seed, args.first_seed + args.seeds):
        clean = synthetic.blob_rect_image(args.size, args.size, 100 + s)
        noisy = synthetic.gaussian_noisy(clean, args.sigma / 255, 200 + s).astype(np.float64)
        row = {"seed": s, "psnr_noisy": psnr(noisy, clean)}
        cfg = TrainConfig(seed=s)
        for impl, name in (() if args.cpu_only else ((1, "simt"), (2, "tf32x3"), (3, "f16x3"))):
            eng = Engine(args.size, args.size, cfg, conv_impl=impl)
            out, r, hist, _, _ = eng.fit_host(np.ascontiguousarray(noisy))
            eng.close()
            row[name] = psnr(out, clean)
            row[name + "_epochs"] = r.epochs_run
        if not args.no_cpu:
            t = time.time()
            ref = o.fit_denoise(noisy, seed=s)
            row["cpu"] = psnr(ref.denoised, clean)
            row["cpu_epochs"] = ref.epochs_run
            row["cpu_s"] = time.time() - t
        rows.append(row)
        print(json.dumps(row), flush=True)
    keys = ([] if args.cpu_only else ["simt", "tf32x3", "f16x3"]) + ([] if args.no_cpu else ["cpu"])
    print(json.dumps({"mean": {k: float(np.mean([r[k] for r in rows])) for k in keys}}))


if __name__ == "__main__":
    main()
