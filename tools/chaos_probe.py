"""How chaotic is the full fit?  Runs the CPU oracle on one image several
times, each with the initial weights perturbed by one ulp in a few random
entries, and reports the spread of final PSNR and stop epochs.  This sizes
what "PSNR within 0.1 dB" can mean at a given image size.

    python tools/chaos_probe.py --size 64 --runs 4
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import n2f_oracle as o  # noqa: E402
from paper_2108_10209_b200 import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=64)
    ap.add_argument("--runs", type=int, default=4)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--rel-noise", type=float, default=0.0,
                    help="instead of 1-ulp nudges, multiply every weight by (1 + N(0, rel_noise))")
    args = ap.parse_args()
    clean = synthetic.blob_rect_image(args.size, args.size, 100 + args.seed)
    noisy = synthetic.gaussian_noisy(clean, 25 / 255, 200 + args.seed).astype(np.float64)
    rng = np.random.default_rng(1)
    out = []
    for r in range(args.runs):
        net = o.init_net(args.seed)
        if r > 0 and args.rel_noise > 0:
            for w in net.weights:
                w *= (1 + rng.normal(0, args.rel_noise, w.shape)).astype(np.float32)
        elif r > 0:  # nudge 8 random weights of L8 by one ulp
            w = net.weights[7].reshape(-1)
            idx = rng.integers(0, w.size, 8)
            w[idx] = np.nextafter(w[idx], np.float32(np.inf))
        res = o.fit_denoise(noisy, seed=args.seed, net=net)
        p = 10 * np.log10(1.0 / np.mean((res.denoised - clean) ** 2))
        out.append(p)
        print(json.dumps({"run": r, "psnr": p, "epochs": res.epochs_run}), flush=True)
    print(json.dumps({"size": args.size, "psnr_spread_db": float(np.max(out) - np.min(out)),
                      "psnr_std_db": float(np.std(out))}))


if __name__ == "__main__":
    main()
