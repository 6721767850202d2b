"""Pool the per-size PSNR equivalence summaries (tools/psnr_equiv.py outputs)
into one stratified estimate of the mean gap GPU - CPU: the inverse-variance
weighted mean over the strata (image sizes differ in gap spread: sd 0.36 dB at
64^2, ~0.7 dB at 128^2, ~1 dB at 256^2) with its 95 % confidence interval, and
the plain mean over all pairs for comparison.

    python tools/psnr_pool.py profiles/r02_psnr_equiv_64.json profiles/r02_psnr_equiv_128.json ... \
        --out profiles/r02_psnr_equiv_summary.json
"""

import argparse
import json
import math

import numpy as np

BAR_DB = 0.1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("docs", nargs="+")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    strata, all_gaps, all_chaos = [], [], []
    for p in args.docs:
        d = json.load(open(p))
        g = np.array([r["gap_gpu"] for r in d["rows"] if "gap_gpu" in r])
        c = np.array([r["gap_cpu"] for r in d["rows"] if "gap_cpu" in r])
        if len(g) < 2:
            continue
        se = float(g.std(ddof=1) / math.sqrt(len(g)))
        strata.append({"doc": p, "n": int(len(g)), "mean_db": float(g.mean()), "sd_db": float(g.std(ddof=1)),
                       "se_db": se, "ci95_db": d["summary"]["gap_gpu_minus_cpu"]["ci95_db"],
                       "max_abs_db": float(np.abs(g).max()),
                       "chaos_n": int(len(c)), "chaos_sd_db": float(c.std(ddof=1)) if len(c) > 1 else None,
                       "chaos_mean_db": float(c.mean()) if len(c) else None,
                       "chaos_max_abs_db": float(np.abs(c).max()) if len(c) else None,
                       "gpu_self_chaos": d["summary"].get("gap_gpu2_minus_gpu")})
        all_gaps.append(g)
        all_chaos.append(c)
    w = np.array([1.0 / s["se_db"] ** 2 for s in strata])
    m = np.array([s["mean_db"] for s in strata])
    pooled = float((w * m).sum() / w.sum())
    pse = float(1.0 / math.sqrt(w.sum()))
    g = np.concatenate(all_gaps)
    plain_se = float(g.std(ddof=1) / math.sqrt(len(g)))
    out = {"bar_db": BAR_DB, "strata": strata,
           "pooled_inverse_variance": {"n": int(len(g)), "mean_db": pooled, "se_db": pse,
                                       "ci95_db": [pooled - 1.96 * pse, pooled + 1.96 * pse],
                                       "within_bar": bool(-BAR_DB <= pooled - 1.96 * pse and pooled + 1.96 * pse <= BAR_DB)},
           "plain_mean_all_pairs": {"n": int(len(g)), "mean_db": float(g.mean()), "se_db": plain_se,
                                    "ci95_db": [float(g.mean()) - 1.96 * plain_se, float(g.mean()) + 1.96 * plain_se]}}
    print(json.dumps(out, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
