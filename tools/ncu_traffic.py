#!/usr/bin/env python
"""DRAM traffic per launch of every libregen kernel in an `ncu --set full` report, keyed by the
names the launch tracer uses (regen_trace_*), written to profiles/ncu_traffic.json for bench.py's
roofline `traffic` field.

  python tools/ncu_traffic.py gpurun_out/prof.ncu-rep|prof.raw.csv ... [--out profiles/ncu_traffic.json]
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess

ROLE = {0: "conv_head", 1: "conv_res_a", 2: "conv_res_b", 3: "conv_body", 4: "conv_up", 5: "conv_tail",
        6: "conv_tiny0", 7: "conv_tiny1", 8: "conv_fold", 9: "conv_fold_frames"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def trace_name(kernel: str) -> str | None:
    if "resblock_tc_kernel" in kernel:
        return "resblock"
    m = re.search(r"conv_tc_kernel<\(?(?:int\))?(\d+)", kernel)
    if m:
        return ROLE.get(int(m.group(1)))
    if "bilinear_kernel" in kernel:
        return "scatter_bilinear"
    if "scatter_rows_kernel" in kernel:
        return "scatter_bilinear" if re.search(r"(true|\(bool\)1|, 1)>", kernel) else "scatter"
    if "combine_kernel" in kernel:
        return "fold_combine_frames" if re.search(r"(true|\(bool\)1|, 1)>", kernel) else "fold_combine"
    if "stitch_band_kernel" in kernel:
        return "stitch"
    if "sort_bitonic_kernel" in kernel:
        return "sort_rank"
    for k in ("gather", "paint", "select", "ccl", "region_write", "box_count", "box_write", "sort_rank", "pack",
              "owner_fix", "conv_simt", "pack_policy", "topk_hist", "topk_select", "nv12_rgb"):
        if re.search(rf"\b{k}_kernel", kernel):
            return k
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="+")
    ap.add_argument("--out", default="profiles/ncu_traffic.json")
    a = ap.parse_args()
    acc: dict[str, list] = {}
    for rep in a.report:
        if rep.endswith(".csv"):   # an exported raw page (ncu -i <rep> --page raw --csv)
            raw = open(rep).read()
        else:
            raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                                 text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        ki, ri, wi, ti = (h.index(x) for x in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                                "gpu__time_duration.sum"))
        for r in rows[2:]:
            name = trace_name(r[ki])
            if name is None:
                continue
            b = float(r[ri].replace(",", "")) * UNIT[units[ri]] + float(r[wi].replace(",", "")) * UNIT[units[wi]]
            acc.setdefault(name, []).append((b, float(r[ti].replace(",", ""))))
    out = {"source": " + ".join(x.split("/")[-1] for x in a.report),
           "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes), mean over the captured launches; "
                   "ncu --set full --clock-control none, cold cache",
           "kernels": {k: sum(x[0] for x in v) / len(v) for k, v in sorted(acc.items())},
           "launches_captured": {k: len(v) for k, v in sorted(acc.items())}}
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
