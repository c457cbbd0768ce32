#!/usr/bin/env python
"""Per-kernel device times of the hot path (analysis aid, NOT a bench number): runs the bench
workload's pipeline a few times under torch.profiler (CUPTI activity tracing) and prints the mean
duration of every libregen kernel, in launch order of one step.

  python tools/kernel_times.py [--config c2] [--steps 5]
"""
from __future__ import annotations

import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2407_16990_b200 as rg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    wl = synth.CONFIGS[a.config]
    imp = torch.from_numpy(synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 0, "blobs")).cuda()
    fr = torch.from_numpy(synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, 0)).cuda()
    w = synth.sr_weights(wl.sr, 0)
    p = rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=wl.bin_w, bin_h=wl.bin_h, max_bins=wl.max_bins,
                    partition_mb=wl.partition_mb, scale=wl.sr.scale, channels=wl.sr.channels,
                    n_resblocks=wl.sr.n_resblocks, weights=w, bf16=wl.sr.bf16)
    for _ in range(3):
        p.run(imp, fr)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(a.steps):
            p.run(imp, fr)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    per = collections.OrderedDict()
    for e in evs:
        name = e.name
        if "FillFunctor" in name or "Memset" in name or "Memcpy" in name:
            continue
        per.setdefault(name, []).append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
    tot = 0.0
    for name, ts in per.items():
        n_per_step = len(ts) / a.steps
        mean = sum(ts) / len(ts)
        tot += mean * n_per_step
        print(f"{mean:9.1f} us x{n_per_step:4.1f}  {name[:110]}")
    print(f"{tot:9.1f} us  total kernel time per step (serialised sum)")


if __name__ == "__main__":
    main()
