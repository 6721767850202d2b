"""FP16x3 range trace over full default fits (VERDICT r01 "next" #2): for the
BASELINE configs (2: 512^2 sigma 50, 3: 1024^2 microscopy, 5: 4096^2), the
per-epoch max |x * 2^e| of every operand-pair slot (tensor class x layer)
that the engine's range guard records (Engine.range_history), with the
headroom to the guard's 2^15 limit and to fp16's 65504.

    python tools/range_trace.py --configs 2 3 5 --out profiles/r02_range_trace.json
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2108_10209_b200 import Engine, TrainConfig, synthetic  # noqa: E402

CLASSES = ("act", "val_act", "grad", "weight")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[2, 3, 5])
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    doc = {"what": "per-epoch max |x * 2^e| of the FP16x3 operand pairs per (class, layer) over full "
                   "default fits (TrainConfig(seed=0)); classes: act = training layer outputs, val_act "
                   "= validation layer outputs, grad = gradients at a layer's pre-activation, weight = "
                   "the tcgen05 layers' weights; e = 8 for act/weight, ceil(log2 P) + 8 for grad",
           "limit_guard": 2.0 ** 15, "fp16_max": 65504.0, "fits": []}
    for cfg in args.configs:
        noisy, _ = synthetic.config_image(cfg, 0)
        h, w = noisy.shape
        eng = Engine(h, w, TrainConfig(seed=0))
        t = time.time()
        out, r, hist, _, _ = eng.fit_host(np.ascontiguousarray(noisy))
        rh = eng.range_history()  # [epochs, 4, 9]
        eng.close()
        peak = rh.max(axis=0)
        slots = {}
        for c, name in enumerate(CLASSES):
            for li in range(9):
                if peak[c, li] > 0:
                    col = rh[:, c, li]
                    slots[f"{name}_L{li + 1}"] = {
                        "max": float(peak[c, li]), "epoch_of_max": int(np.argmax(col)) + 1,
                        "first": float(col[0]), "last": float(col[-1]),
                        "headroom_bits_to_guard": float(np.log2(2.0 ** 15 / peak[c, li]))}
        fit = {"config": cfg, "shape": [h, w], "epochs": int(r.epochs_run), "seconds": time.time() - t,
               "overall_max": float(peak.max()),
               "min_headroom_bits_to_guard": float(np.log2(2.0 ** 15 / peak.max())),
               "slots": slots,
               "per_epoch_max_by_class": {name: rh[:, c, :].max(axis=1).round(4).tolist()
                                          for c, name in enumerate(CLASSES)}}
        doc["fits"].append(fit)
        print(json.dumps({k: v for k, v in fit.items() if k not in ("slots", "per_epoch_max_by_class")}),
              flush=True)
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
