"""Per-epoch divergence between the CPU oracle and the GPU engine over a
bounded fit (no early stop): validation score and weights after each epoch.

    python tools/trajectory_diff.py --size 64 --epochs 30
"""

import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402

from n2f_testutil import arena_to_layers, norm_rel  # noqa: E402
from oracle import n2f_oracle as o  # noqa: E402
from paper_2108_10209_b200 import Engine, TrainConfig, _lib, synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=64)
    ap.add_argument("--epochs", type=int, default=30)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impls", default="1,2")
    args = ap.parse_args()
    s = args.seed
    clean = synthetic.blob_rect_image(args.size, args.size, 100 + s)
    noisy = synthetic.gaussian_noisy(clean, 25 / 255, 200 + s).astype(np.float64)
    n32 = o.normalize(noisy)[0].astype(np.float32)
    pairs = o.training_pairs(n32)
    shapes = o.layer_shapes()
    impls = [int(v) for v in args.impls.split(",")]
    engs = {}
    for impl in impls:
        eng = Engine(args.size, args.size, TrainConfig(seed=s, max_epochs=args.epochs + 5),
                     use_graph=False, conv_impl=impl)
        _lib.call("n2f_ctx_prepare", eng.handle, np.ascontiguousarray(noisy).ctypes.data,
                  _lib.N2F_F64, None, 1)
        engs[impl] = eng
    net = o.init_net(s)
    n = C.c_int64()
    _lib.call("n2f_ctx_param_count", engs[impls[0]].handle, C.byref(n))
    arena = np.empty(n.value, np.float32)
    for e in range(1, args.epochs + 1):
        for a, b in pairs:
            z, cache = o.net_forward(net, a, keep=True)
            _, gz = o.bce_logits(z, b)
            o.net_step(net, o.net_backward(net, cache, gz), 1e-3)
        ref_out = o.predict(net, n32)
        ref_score = o.val_score(ref_out, n32)
        row = {"epoch": e, "cpu_score": ref_score}
        for impl, eng in engs.items():
            for k in range(4):
                _lib.call("n2f_ctx_step", eng.handle, k, None)
            out = np.empty(noisy.size, np.float32)
            sc = C.c_double()
            _lib.call("n2f_ctx_validate", eng.handle, out.ctypes.data, C.byref(sc))
            _lib.call("n2f_ctx_get_arena", eng.handle, 0, arena.ctypes.data)
            layers = arena_to_layers(arena, shapes)
            werr = max(norm_rel(w, rw) for (w, _), rw in zip(layers, net.weights))
            row[f"i{impl}_score_rel"] = (sc.value - ref_score) / ref_score
            row[f"i{impl}_out_rel"] = norm_rel(out.reshape(noisy.shape), ref_out)
            row[f"i{impl}_w_rel"] = werr
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
