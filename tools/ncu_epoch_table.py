"""Per-kernel-class ncu table of one host-loop epoch at 512^2 (VERDICT r01
row N1): every launch of `tools/ncu_target.py 1` under `ncu --set full`,
labelled by its place in the epoch (L1 forward, L2..L8 forward / dgrad /
wgrad, Adam, validation, stop, window mean), with duration, tensor-pipe
activity, DRAM bytes and achieved GB/s, and algorithmic TFLOP/s for the
convolutions.

    ncu -i epoch.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_epoch_table.py raw.csv[.gz] --out profiles/r02_ncu_epoch512.json
"""

import argparse
import csv
import gzip
import io
import json
import re

CIN = [1, 32, 32, 64, 64, 128, 128, 256, 256]
COUT = [32, 32, 64, 64, 128, 128, 256, 256, 1]
H = W = 512
PT = H * W // 2
PV = H * W

M_DUR = "gpu__time_duration.sum"
M_TENSOR = "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"
M_TMEM = "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
M_TCSMEM = "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"
M_RD = "dram__bytes_read.sum"
M_WR = "dram__bytes_write.sum"
M_ISSUE = "sm__inst_issued.avg.pct_of_peak_sustained_active"
M_CLK = "gpc__cycles_elapsed.avg.per_second"


def conv_flop(P, li):
    return 2.0 * P * COUT[li] * 9 * CIN[li]


def read_raw(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        rows = list(csv.reader(io.StringIO(f.read())))
    head, units = rows[0], rows[1]

    def norm(c):  # "TPC.TriageCompute.sm__pipe_..." -> "sm__pipe_..."
        parts = c.split(".")
        for i, q in enumerate(parts):
            if "__" in q:
                return ".".join(parts[i:])
        return c

    head = [norm(c) for c in head]
    out = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        d["_units"] = dict(zip(head, units))
        out.append(d)
    return out


def num(d, key):
    v = d.get(key, "")
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    u = d["_units"].get(key, "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
             "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(u, 1)
    return x * scale


def label_epoch(kernels):
    """Assign labels to one host-loop epoch's launches (fit prep first)."""
    names = [k["Kernel Name"] for k in kernels]
    labels = [None] * len(kernels)
    i = 0
    # skip prep up to the first training-step forward of L1
    while i < len(names) and "k_conv_first" not in names[i]:
        labels[i] = "prep:" + re.sub(r"\(.*", "", names[i]).split("::")[-1]
        i += 1
    for step in range(4):
        seq = [("fwd", 0, "k_conv_first")] + [("fwd", li, "k_conv3x3_dy") for li in range(1, 8)]
        for li in range(7, 0, -1):
            seq += [("wgrad", li, "k_wgrad3x3_tc"), ("dgrad", li, "k_conv3x3_dy")]
        seq += [("wgrad", 0, "k_wgrad_first"), ("adam", -1, "k_adam"),
                ("transpose", -1, "k_transpose_pairs")]
        for kind, li, pat in seq:
            assert pat in names[i], (i, names[i], pat)
            labels[i] = (f"step{step}", kind, li)
            i += 1
    seq = [("val", 0, "k_conv_first")] + [("val", li, "k_conv3x3_dy") for li in range(1, 8)] + \
          [("stop", -1, "k_stop")]
    for kind, li, pat in seq:
        assert pat in names[i], (i, names[i], pat)
        labels[i] = ("val", kind, li)
        i += 1
    while i < len(names):
        labels[i] = "tail:" + re.sub(r"\(.*", "", names[i]).split("::")[-1]
        i += 1
    return labels


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    ks = read_raw(args.raw)
    labels = label_epoch(ks)
    classes = {}
    for k, lab in zip(ks, labels):
        if isinstance(lab, str):
            key = lab
            flop = 0.0
        else:
            where, kind, li = lab
            key = f"{kind} L{li + 1}" if li >= 0 else kind
            if kind in ("fwd", "dgrad", "wgrad"):
                flop = conv_flop(PT, li)
            elif kind == "val":
                flop = conv_flop(PV, li)
            else:
                flop = 0.0
            if kind in ("fwd", "val") and li == 7:
                key += " (+ fused L9 head)"
        c = classes.setdefault(key, {"launches": 0, "kernel": re.sub(r"\(.*", "", k["Kernel Name"])[:80],
                                     "dur_s": 0.0, "dram_bytes": 0.0, "flop": 0.0, "tensor_pct": [],
                                     "tmem_pct": [], "issue_pct": [], "tc_smem_pct": []})
        c["launches"] += 1
        c["dur_s"] += num(k, M_DUR) or 0.0
        c["dram_bytes"] += (num(k, M_RD) or 0.0) + (num(k, M_WR) or 0.0)
        c["flop"] += flop
        for m, f in ((M_TENSOR, "tensor_pct"), (M_TMEM, "tmem_pct"), (M_ISSUE, "issue_pct"),
                     (M_TCSMEM, "tc_smem_pct")):
            v = num(k, m)
            if v is not None:
                c[f].append(v)
    table = {}
    total = sum(c["dur_s"] for c in classes.values())
    for key, c in classes.items():
        n = c["launches"]
        row = {"kernel": c["kernel"], "launches": n, "us_per_launch": 1e6 * c["dur_s"] / n,
               "share_of_epoch": c["dur_s"] / total if total else None,
               "dram_MB_per_launch": c["dram_bytes"] / n / 1e6,
               "dram_GBps": c["dram_bytes"] / c["dur_s"] / 1e9 if c["dur_s"] else None}
        for f in ("tensor_pct", "tmem_pct", "issue_pct", "tc_smem_pct"):
            if c[f]:
                row[f] = sum(c[f]) / len(c[f])
        if c["flop"]:
            row["algorithmic_TFLOPs"] = c["flop"] / c["dur_s"] / 1e12
        table[key] = row
    doc = {"what": "ncu --set full --clock-control none, one host-loop epoch of the 512^2 config-2 image "
                   "(tools/ncu_target.py 1); per kernel class: mean duration, tensor-pipe activity "
                   "(sm__pipe_tensor_cycles_active_realtime), tensor-memory pipe activity "
                   "(sm__mem_tensor_cycles_active), issue slots, DRAM bytes "
                   "and achieved GB/s; algorithmic TFLOP/s = 2*P*Cout*9*Cin per launch / duration. "
                   "ncu serialises and cold-starts each launch, so durations are per-kernel upper bounds.",
           "epoch_kernel_time_ms": 1e3 * total, "classes": table}
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)
    for key, r in table.items():
        print(f"{key:28s} n={r['launches']:2d} {r['us_per_launch']:8.1f} us  "
              f"pipe_tensor={r.get('tensor_pct', float('nan')):5.1f}% mem_tensor={r.get('tmem_pct', float('nan')):5.1f}% "
              f"issue={r.get('issue_pct', float('nan')):5.1f}% dram={r['dram_GBps'] or 0:6.0f} GB/s "
              f"TF/s={r.get('algorithmic_TFLOPs', float('nan')):6.1f}")


if __name__ == "__main__":
    main()
