"""Merge per-seed PSNR parity rows (tools/psnr_parity.py output) into one
profile with the summary statistics used in DESIGN.md section 4.

    python tools/psnr_merge.py --base profiles/r01_psnr_parity_256.json \
        --rows a.jsonl b.jsonl ... --out profiles/r01_psnr_parity_256_v2.json

Rows from separate GPU (--no-cpu) and CPU (--cpu-only) runs of the same seed
are joined on "seed"; "cpu" is stored as "cpu_oracle" as in the base file.
"""

import argparse
import json

import numpy as np

IMPLS = ("simt", "tf32x3", "f16x3")


def summarise(rows):
    c = np.array([r["cpu_oracle"] for r in rows])
    out = {"cpu_oracle": {"mean": float(c.mean()), "std": float(c.std(ddof=1))}}
    for k in IMPLS:
        v = np.array([r[k] for r in rows])
        d = v - c
        out[k] = {"mean": float(v.mean()), "std": float(v.std(ddof=1)),
                  "mean_diff_vs_cpu": float(d.mean()),
                  "se_diff": float(d.std(ddof=1) / np.sqrt(len(d))),
                  "max_abs_diff": float(np.abs(d).max())}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--base", required=True)
    ap.add_argument("--rows", nargs="+", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--what", default=None)
    args = ap.parse_args()
    base = json.load(open(args.base))
    by_seed = {r["seed"]: dict(r) for r in base["rows"]}
    for path in args.rows:
        for line in open(path):
            line = line.strip()
            if not line.startswith("{") or '"seed"' not in line:
                continue
            r = json.loads(line)
            if "cpu" in r:
                r["cpu_oracle"] = r.pop("cpu")
            by_seed.setdefault(r["seed"], {}).update(r)
    rows = [by_seed[s] for s in sorted(by_seed)
            if all(k in by_seed[s] for k in IMPLS + ("cpu_oracle",))]
    missing = sorted(set(by_seed) - {r["seed"] for r in rows})
    doc = {"what": args.what or base["what"], "n_seeds": len(rows),
           "incomplete_seeds": missing, "rows": rows, "summary": summarise(rows)}
    json.dump(doc, open(args.out, "w"), indent=1)
    print(json.dumps(doc["summary"], indent=1))


if __name__ == "__main__":
    main()
