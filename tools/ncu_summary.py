"""Summarise ncu --set full reports into JSON (key SOL / occupancy numbers,
tensor-pipe activity and DRAM bytes per launch).

    python tools/ncu_summary.py out.json label=path.ncu-rep [label=path ...]
"""

import csv
import io
import json
import subprocess
import sys

DETAILS = ["SM Frequency", "Elapsed Cycles", "Duration", "DRAM Throughput", "L2 Cache Throughput",
           "Compute (SM) Throughput", "L2 Hit Rate", "Registers Per Thread",
           "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Issue Slots Busy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum"]


def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep):
    kernels = []
    rows = page(rep, "details")
    h = rows[0]
    by_id = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = by_id.setdefault(d["ID"], {"kernel": d["Kernel Name"][:100]})
        if d["Metric Name"] in DETAILS and d["Metric Name"] not in k:
            k[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'
    raw = page(rep, "raw")
    rh, units = raw[0], raw[1]
    # raw column names may carry a section prefix ("TPC.TriageCompute.<metric>")
    rh = [c.split(".", 2)[-1] if c.count(".") >= 3 and not c.startswith(("dram", "gpu", "sm", "l1tex", "lts"))
          else c for c in rh]
    for i, r in enumerate(raw[2:]):
        d = dict(zip(rh, r))
        k = by_id.get(d.get("ID"), None)
        if k is None:
            continue
        for name in RAW:
            if name in d:
                k[name] = f"{d[name]} {units[rh.index(name)]}"
    return list(by_id.values())


def main():
    out = sys.argv[1]
    res = {}
    for arg in sys.argv[2:]:
        label, path = arg.split("=", 1)
        res[label] = summarise(path)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
