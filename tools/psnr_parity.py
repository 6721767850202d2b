"""GPU side of the PSNR equivalence study: full default fits of the engine on
the seeded images of tools/psnr_equiv_cpu.py (128^2 blob+rect, clean seed
100+s, noise seed 200+s, sigma 25/255, TrainConfig(seed=s)), one JSON row per
seed.  tools/psnr_equiv.py joins these rows with the CPU reference rows.

    python tools/psnr_parity.py --size 128 --seeds 0-149 --out gpurun_out/psnr_gpu.jsonl
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2108_10209_b200 import TrainConfig, synthetic, train_single_channel  # noqa: E402


def psnr(a, b):
    return 10 * np.log10(1.0 / np.mean((np.asarray(a, np.float64) - b) ** 2))


def parse_seeds(s):
    out = []
    for part in s.split(","):
        a, _, b = part.partition("-")
        out.extend(range(int(a), int(b or a) + 1))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=128)
    ap.add_argument("--seeds", default="0-149")
    ap.add_argument("--sigma", type=float, default=25.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--image", default="study", choices=["study", "config1"])
    ap.add_argument("--perturb", type=float, default=0.0,
                    help="kind gpu2: the engine's own chaos partner, the same fit of the image "
                         "multiplied by (1 + N(0, perturb)) per pixel (1e-7: last-bit changes of the "
                         "normalised float32 image); PSNR is still taken against the clean image")
    args = ap.parse_args()
    sink = open(args.out, "a") if args.out else None
    for s in parse_seeds(args.seeds):
        if args.image == "config1":  # BASELINE.json config 1 (256^2, sigma 25/255)
            noisy, clean = synthetic.config_image(1, s)
            noisy, args.size = noisy.astype(np.float64), 256
        else:
            clean = synthetic.blob_rect_image(args.size, args.size, 100 + s)
            noisy = synthetic.gaussian_noisy(clean, args.sigma / 255, 200 + s).astype(np.float64)
        if args.perturb > 0:
            noisy = noisy * (1 + np.random.default_rng(10_000 + s).normal(0, args.perturb, noisy.shape))
        t = time.time()
        r = train_single_channel(noisy, TrainConfig(seed=s))
        row = {"kind": "gpu2" if args.perturb > 0 else "gpu", "seed": s, "size": args.size, "image": args.image, "psnr": float(psnr(r.denoised, clean)),
               "psnr_noisy": float(psnr(noisy, clean)), "epochs": r.epochs_run,
               "stop": r.stop_reason, "s": time.time() - t}
        print(json.dumps(row), flush=True)
        if sink:
            sink.write(json.dumps(row) + "\n")
            sink.flush()


if __name__ == "__main__":
    main()
