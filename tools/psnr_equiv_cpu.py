"""CPU side of the PSNR equivalence study (VERDICT r01 "next" #1).

Runs full default fits of the STOCK reference (`noise2fast.trainer.
train_single_channel`, imported from /root/reference/pkg/src in this
container) on the seeded 128^2 blob+rect images of tools/psnr_parity.py
(clean seed 100+s, noise seed 200+s, sigma 25/255, TrainConfig(seed=s)):

  kind "cpu"  : the unmodified reference fit;
  kind "cpu2" : the same fit with every initial weight multiplied by
                (1 + N(0, 1e-7)) -- the reference's own chaos partner
                (build_network wrapped, everything else stock).

One JSON row per (kind, seed) is appended to --out; finished rows are skipped
on restart, so the job is resumable.  A pool of single-BLAS-thread workers
runs the fits (the reference is single-threaded per fit apart from BLAS).

    python tools/psnr_equiv_cpu.py --out profiles/r02_psnr_equiv_cpu.jsonl \
        --seeds 0-149 --kinds cpu2,cpu --workers 6
"""

import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor, as_completed

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"


def _worker_init():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/n2f_numba_cache")
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REPO)


def _fit(kind: str, seed: int, size: int, sigma: float, image: str = "study"):
    import numpy as np
    from noise2fast import model, trainer

    from paper_2108_10209_b200 import synthetic

    if image == "config1":  # BASELINE.json config 1 (256^2, sigma 25/255), image seed = fit seed
        noisy, clean = synthetic.config_image(1, seed)
        noisy, size = noisy.astype(np.float64), 256
    else:
        clean = synthetic.blob_rect_image(size, size, 100 + seed)
        noisy = synthetic.gaussian_noisy(clean, sigma / 255, 200 + seed).astype(np.float64)
    orig = model.build_network
    if kind == "cpu2":
        rng = np.random.default_rng(10_000 + seed)

        def perturbed(in_ch, s, lr=0.001):
            net = orig(in_ch, s, lr=lr)
            for layer in net.layers:
                w = layer.weights
                w *= (1 + rng.normal(0, 1e-7, w.shape)).astype(w.dtype)
            return net

        model.build_network = perturbed
    try:
        t = time.time()
        res = trainer.train_single_channel(noisy, trainer.TrainConfig(seed=seed))
        dt = time.time() - t
    finally:
        model.build_network = orig
    p = 10 * np.log10(1.0 / np.mean((res.denoised - clean) ** 2))
    return {"kind": kind, "seed": seed, "size": size, "image": image, "psnr": float(p),
            "psnr_noisy": float(10 * np.log10(1.0 / np.mean((noisy - clean) ** 2))),
            "epochs": res.epochs_run, "stop": res.stop_reason, "s": dt}


def _parse_seeds(s: str):
    out = []
    for part in s.split(","):
        a, _, b = part.partition("-")
        out.extend(range(int(a), int(b or a) + 1))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--seeds", default="0-149")
    ap.add_argument("--kinds", default="cpu2,cpu")
    ap.add_argument("--size", type=int, default=128)
    ap.add_argument("--sigma", type=float, default=25.0)
    ap.add_argument("--workers", type=int, default=6)
    ap.add_argument("--image", default="study", choices=["study", "config1"])
    ap.add_argument("--blas-threads", type=int, default=1)
    args = ap.parse_args()
    if args.image == "config1":
        args.size = 256
    done = set()
    if os.path.exists(args.out):
        for line in open(args.out):
            if line.startswith("{"):
                r = json.loads(line)
                if r.get("image", "study") == args.image:
                    done.add((r["kind"], r["seed"], r["size"]))
    kinds = args.kinds.split(",")
    jobs = [(k, s) for s in _parse_seeds(args.seeds) for k in kinds
            if (k, s, args.size) not in done]
    print(f"{len(jobs)} fits to run", flush=True)
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = str(args.blas_threads)
    with ProcessPoolExecutor(args.workers, initializer=_worker_init) as ex:
        futs = [ex.submit(_fit, k, s, args.size, args.sigma, args.image) for k, s in jobs]
        with open(args.out, "a") as f:
            for fu in as_completed(futs):
                row = fu.result()
                f.write(json.dumps(row) + "\n")
                f.flush()
                print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
