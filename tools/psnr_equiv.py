"""PSNR equivalence study (VERDICT r01 "next" #1): join the GPU engine's full
fits (tools/psnr_parity.py rows, kind "gpu") with the stock reference's fits
of the same seeded images (tools/psnr_equiv_cpu.py rows: kind "cpu" = the
unmodified reference, kind "cpu2" = the reference with 1e-7 relative init
noise) and report

  gap_gpu = PSNR(GPU) - PSNR(CPU)     the engine against the reference
  gap_cpu = PSNR(CPU') - PSNR(CPU)    the reference against itself (chaos)

per seed, with the mean, its standard error and 95 % confidence interval
(Student t), the spread of both gap distributions, and a two-sample
comparison of them.  The north_star bar is met when the 95 % CI of the mean
gap_gpu lies inside +-0.1 dB.

    python tools/psnr_equiv.py --gpu profiles/r02_psnr_equiv_gpu_128.jsonl \
        --cpu profiles/r02_psnr_equiv_cpu.jsonl --out profiles/r02_psnr_equiv_128.json
"""

from __future__ import annotations

import argparse
import json
import math

import numpy as np

BAR_DB = 0.1


def load(paths, size=None, image="study"):
    rows = {}
    for p in paths:
        for line in open(p):
            line = line.strip()
            if not line.startswith("{"):
                continue
            r = json.loads(line)
            if size is not None and r.get("size") != size:
                continue
            if r.get("image", "study") != image:
                continue
            rows[(r["kind"], r["seed"])] = r
    return rows


def load_r01_cpu(path, rows, size):
    """CPU rows of a round-1 profile (tools/psnr_merge.py format): full fits of
    the oracle port, which is bitwise the stock reference on one epoch with the
    same BLAS (tests/golden).  Only seeds without a stock-reference row."""
    n = 0
    for r in json.load(open(path))["rows"]:
        if "cpu_oracle" in r and ("cpu", r["seed"]) not in rows:
            rows[("cpu", r["seed"])] = {"kind": "cpu", "seed": r["seed"], "size": size,
                                        "psnr": r["cpu_oracle"], "psnr_noisy": r["psnr_noisy"],
                                        "epochs": r["cpu_epochs"], "port": True}
            n += 1
    return n


def t95(df: int) -> float:
    try:
        from scipy import stats

        return float(stats.t.ppf(0.975, df))
    except Exception:
        return 1.96


def describe(d: np.ndarray) -> dict:
    n = len(d)
    if n == 0:
        return {"n": 0}
    mean = float(d.mean())
    sd = float(d.std(ddof=1)) if n > 1 else float("nan")
    se = sd / math.sqrt(n) if n > 1 else float("nan")
    h = t95(n - 1) * se if n > 1 else float("nan")
    return {"n": n, "mean_db": mean, "sd_db": sd, "se_db": se, "ci95_db": [mean - h, mean + h],
            "max_abs_db": float(np.abs(d).max()),
            "within_bar": bool(n > 1 and -BAR_DB <= mean - h and mean + h <= BAR_DB)}


def analyse(rows: dict) -> dict:
    seeds = sorted({s for (k, s) in rows})
    per = []
    for s in seeds:
        c = rows.get(("cpu", s))
        if c is None:
            continue
        e = {"seed": s, "psnr_noisy": c["psnr_noisy"], "cpu": c["psnr"], "cpu_epochs": c["epochs"]}
        if c.get("port"):
            e["port"] = True
        g = rows.get(("gpu", s))
        if g is not None:
            e.update(gpu=g["psnr"], gpu_epochs=g["epochs"], gap_gpu=g["psnr"] - c["psnr"])
        c2 = rows.get(("cpu2", s))
        if c2 is not None:
            e.update(cpu2=c2["psnr"], cpu2_epochs=c2["epochs"], gap_cpu=c2["psnr"] - c["psnr"])
        g2 = rows.get(("gpu2", s))
        if g is not None and g2 is not None:
            e.update(gpu2=g2["psnr"], gpu2_epochs=g2["epochs"], gap_gpu2=g2["psnr"] - g["psnr"])
        per.append(e)
    gg = np.array([e["gap_gpu"] for e in per if "gap_gpu" in e])
    gc = np.array([e["gap_cpu"] for e in per if "gap_cpu" in e])
    # the engine against itself (kind gpu2: last-bit perturbed input), over every seed that has both
    # GPU fits, with or without a CPU row
    g2all = np.array([rows[("gpu2", s)]["psnr"] - rows[("gpu", s)]["psnr"]
                      for (k, s) in rows if k == "gpu2" and ("gpu", s) in rows])
    out = {"bar_db": BAR_DB, "gap_gpu_minus_cpu": describe(gg), "gap_cpu2_minus_cpu": describe(gc),
           "gap_gpu2_minus_gpu": describe(g2all)}
    if len(gg) > 1 and len(gc) > 1:
        try:
            from scipy import stats

            out["sd_ratio_gpu_over_cpu2"] = float(gg.std(ddof=1) / gc.std(ddof=1))
            out["levene_p_equal_spread"] = float(stats.levene(gg, gc).pvalue)
            out["welch_p_equal_mean"] = float(stats.ttest_ind(gg, gc, equal_var=False).pvalue)
        except Exception:
            pass
    cpu = np.array([e["cpu"] for e in per])
    out["cpu_mean_psnr_db"] = float(cpu.mean()) if len(cpu) else None
    out["gpu_mean_psnr_db"] = float(np.mean([e["gpu"] for e in per if "gpu" in e])) if len(gg) else None
    return out, per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpu", nargs="+", required=True)
    ap.add_argument("--cpu", nargs="+", required=True)
    ap.add_argument("--size", type=int, default=128)
    ap.add_argument("--image", default="study", choices=["study", "config1"])
    ap.add_argument("--r01-cpu", default=None,
                    help="round-1 profile whose oracle-port CPU fits fill seeds without a stock-reference row")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.image == "config1":
        args.size = 256
    rows = load(args.gpu + args.cpu, args.size, args.image)
    n_port = load_r01_cpu(args.r01_cpu, rows, args.size) if args.r01_cpu else 0
    summary, per = analyse(rows)
    summary["cpu_rows_from_oracle_port"] = n_port
    images = ("BASELINE config-1 images (256^2, sigma 25/255, image seed = fit seed s)"
              if args.image == "config1" else
              f"{args.size}^2 blob+rect, sigma 25/255, clean seed 100+s, noise seed 200+s")
    doc = {"what": f"full default fit-and-denoise PSNR, {images}, TrainConfig(seed=s); cpu = stock reference "
                   "(noise2fast from /root/reference, 1-2 BLAS threads; rows marked port = the "
                   "oracle port's round-1 fits), cpu2 = stock reference with 1e-7 "
                   "relative init noise, gpu = this engine, gpu2 = this engine on the image times "
                   "(1 + N(0, 1e-7)) per pixel; tools/psnr_equiv.py",
           "summary": summary, "rows": per}
    print(json.dumps(summary, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
