#!/usr/bin/env python
"""Packing-policy / occupy-ratio study on the GPU packer (paper P:1345-1347, P:741-747,
P:1669-1670): for synthetic importance maps of the paper's workloads, run the index path
(regen_select_mbs + regen_pack_regions) with partition limits P in {1 (Block), 2, 3, 4, 7} and the two
region orders (importance density, the paper's choice; max-area-first, the `fig:Puzzle` baseline) and
report, per setting:
  * boxes, bins, fill = box px / bin px, occupy ratio = selected-MB px / box px ("selected MBs
    occupying all enhanced content"), both over the placed boxes;
  * with a fixed bin budget B (capacity mode: boxes that do not fit stay bilinear), the share of the
    selected importance that lands in placed boxes (fig:Puzzle: density order should keep more);
  * the device time of the pack call (box build + sort + Alg. 1 packer), CUDA events, warm.
Analysis aid, not a bench number; writes profiles/r01_packing_study.{json,md}.

  python tools/packing_study.py [--reps 5]
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_16990_b200 as rg  # noqa: E402
import synth  # noqa: E402

WORKLOADS = [
    ("360p 1x30 20% 128^2", dataclasses.replace(synth.CONFIGS["c2"]), 20.0),
    ("720p 2x30 5% 128^2", dataclasses.replace(synth.CONFIGS["c5"]), 5.0),
    ("720p 2x30 25% 128^2", dataclasses.replace(synth.CONFIGS["c5"], pct=25.0), 25.0),
]


def run(wl, imp_d, imp_h, P, order, max_bins, reps):
    p = rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=wl.bin_w, bin_h=wl.bin_h, max_bins=max_bins,
                    partition_mb=P, scale=wl.sr.scale, channels=16, n_resblocks=0,
                    weights=synth.sr_weights(synth.SRConfig(wl.sr.scale, 16, 0, 1.0, True), 0), bf16=True,
                    order=order)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(reps + 1):
        p.select(imp_d)
        torch.cuda.synchronize()
        e0.record()
        p.pack_step(imp_d)
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    r = p.host_results()
    assert r["status"] == 0, r["status"]
    bx = r["boxes"]
    placed = bx["bin"] >= 0
    box_px = int((bx["w"][placed].astype(np.int64) * bx["h"][placed]).sum())
    owner = r["owner"]
    sel = r["sel"].astype(bool)
    sel_px = int((owner >= 0).sum()) * 256
    imp_sel = float(imp_h[sel].astype(np.float64).sum())
    imp_kept = float(imp_h[owner >= 0].astype(np.float64).sum())
    nb = r["num_bins"]
    return {"boxes": int(r["num_boxes"]), "placed": int(placed.sum()), "bins": nb,
            "fill_box_over_bin": box_px / max(nb * wl.bin_w * wl.bin_h, 1),
            "occupy_sel_over_box": sel_px / max(box_px, 1),
            "importance_kept": imp_kept / max(imp_sel, 1e-30),
            "pack_ms": float(np.median(ts))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "profiles"))
    a = ap.parse_args()
    torch.cuda.set_device(0)
    out = []
    for name, wl, pct in WORKLOADS:
        imp_h = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 0)
        imp_d = torch.from_numpy(imp_h).cuda()
        for P in (1, 2, 3, 4, 7):
            for order, oname in ((rg.ORDER_DENSITY, "density"), (rg.ORDER_AREA, "area")):
                open_bins = run(wl, imp_d, imp_h, P, order, wl.max_bins, a.reps)
                # capacity mode: the bin budget of the paper's N at this ratio, i.e. as many bins
                # as the selected MBs would fill without expansion
                cap = max(1, (wl.k * 256 + wl.bin_w * wl.bin_h - 1) // (wl.bin_w * wl.bin_h))
                capped = run(wl, imp_d, imp_h, P, order, cap, 1)
                out.append({"workload": name, "P": P, "order": oname, "open_bins": open_bins,
                            "capacity_bins": cap, "capacity": capped})
                print(name, P, oname, json.dumps(open_bins), "cap", cap, round(capped["importance_kept"], 4),
                      flush=True)
    os.makedirs(a.out_dir, exist_ok=True)
    with open(os.path.join(a.out_dir, "r01_packing_study.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    lines = ["# Packing study (GPU packer, synthetic maps; tools/packing_study.py)", "",
             "fill = placed box px / bin px; occupy = selected-MB px / placed box px (P:1345); kept = share of the "
             "selected importance inside placed boxes when the bin budget is the paper's N = k*256/(H*W) bins "
             "(P:663, expansion not budgeted); pack ms = device time of regen_pack_regions (box build + sort + "
             "Alg. 1), median of warm runs.", "",
             "| workload | P | order | boxes | bins | fill | occupy | pack ms | budget bins | kept (budget) |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in out:
        o, c = r["open_bins"], r["capacity"]
        lines.append(f"| {r['workload']} | {r['P']} | {r['order']} | {o['boxes']} | {o['bins']} | "
                     f"{o['fill_box_over_bin']:.3f} | {o['occupy_sel_over_box']:.3f} | {o['pack_ms']:.3f} | "
                     f"{r['capacity_bins']} | {c['importance_kept']:.3f} |")
    with open(os.path.join(a.out_dir, "r01_packing_study.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
