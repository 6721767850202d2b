"""Golden final PSNRs of the STOCK reference's full default fits, for the GPU
PSNR equivalence test (tests/test_gpu_psnr_equivalence.py).

The fits themselves were run by tools/psnr_equiv_cpu.py (it imports
/root/reference/pkg/src and appends one JSON row per fit to
profiles/r02_psnr_equiv_cpu*.jsonl; ~10 CPU-minutes per 128^2 fit, so they are
not repeated here); this script only collects the kind "cpu" rows into
tests/golden/psnr_reference_fits.json, keyed by image family, size and seed.

    python tests/golden/make_psnr_golden.py
"""

import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    fits = {}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r02_psnr_equiv_cpu*.jsonl"))):
        for line in open(path):
            if not line.startswith("{"):
                continue
            r = json.loads(line)
            if r["kind"] != "cpu":
                continue
            key = f"{r.get('image', 'study')}:{r['size']}"
            fits.setdefault(key, {})[str(r["seed"])] = {
                "psnr": r["psnr"], "psnr_noisy": r["psnr_noisy"], "epochs": r["epochs"]}
    doc = {"what": "final PSNR (dB) of noise2fast.trainer.train_single_channel (stock reference, CPU) with "
                   "TrainConfig(seed=s); 'study:N' = N x N blob+rect image, clean seed 100+s, noise seed "
                   "200+s, sigma 25/255; 'config1:256' = BASELINE config 1 with image seed s",
           "fits": {k: dict(sorted(v.items(), key=lambda kv: int(kv[0]))) for k, v in sorted(fits.items())}}
    out = os.path.join(ROOT, "tests", "golden", "psnr_reference_fits.json")
    with open(out, "w") as f:
        json.dump(doc, f, indent=0)
    print({k: len(v) for k, v in doc["fits"].items()}, "->", out)


if __name__ == "__main__":
    main()
