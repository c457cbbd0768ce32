#!/usr/bin/env python
"""One small run of the bench model (EDSR 8x32 x3, C2 geometry with 2 frames) through every ABI call, for
compute-sanitizer (memcheck / racecheck / synccheck): the C = 32 kernel instances the bench uses
(fused residual block, fused fold + combine, bilinear pass, 8-warp packer path on a noisy map).

  compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_16990_b200 as rg  # noqa: E402
import synth  # noqa: E402

wl = synth.small(synth.CONFIGS["c2"], F=2)
for kind in ("blobs", "noisy"):
    imp = torch.from_numpy(synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 3, kind)).cuda()
    fr = torch.from_numpy(synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, 3)).cuda()
    p = rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=wl.bin_w, bin_h=wl.bin_h, max_bins=wl.max_bins,
                    partition_mb=1 if kind == "noisy" else wl.partition_mb, scale=wl.sr.scale,
                    channels=wl.sr.channels, n_resblocks=wl.sr.n_resblocks,
                    weights=synth.sr_weights(wl.sr, 0), bf16=True)
    out = p.run(imp, fr)                       # regen_enhance_scatter (fused fold)
    p.enhance_owned(fr, out=out)
    p.scatter_bilinear(fr, out=out)
    p.run(imp, fr, fused=False)                # regen_enhance_packed + regen_scatter_blend
    torch.cuda.synchronize()
    r = p.host_results()
    assert r["status"] == 0
    print(kind, "boxes", r["num_boxes"], "bins", r["num_bins"])

# round-2 kernels: the per-bin packer path (> 5000 boxes), the placement policies, the one-pass stitch,
# cross-rank top-N, temporal reuse and NV12 conversion
wl30 = dataclasses.replace(synth.CONFIGS["c2"], partition_mb=1)
imp = torch.from_numpy(synth.importance_maps(wl30.S, wl30.F, wl30.GH, wl30.GW, 5)).cuda()
sr_small = synth.SRConfig(3, 16, 1, 1.0, True)
w_small = synth.sr_weights(sr_small, 0)
p = rg.Pipeline(S=wl30.S, F=wl30.F, W=wl30.W, H=wl30.H, k=wl30.k, bin_w=128, bin_h=128, max_bins=wl30.max_bins,
                partition_mb=1, scale=3, channels=16, n_resblocks=1, weights=w_small)
p.select(imp)
p.pack_step(imp)
print("bins path: boxes", p.host_results()["num_boxes"])
wl4 = synth.small(synth.CONFIGS["c2"], F=4)
imp4 = torch.from_numpy(synth.importance_maps(wl4.S, wl4.F, wl4.GH, wl4.GW, 6, "noisy")).cuda()
for pol, order in ((rg.POLICY_MAXRECT, 0), (rg.POLICY_SKYLINE, 0), (rg.POLICY_SHELF, 2)):
    q = rg.Pipeline(S=wl4.S, F=wl4.F, W=wl4.W, H=wl4.H, k=wl4.k, bin_w=128, bin_h=128, max_bins=64, partition_mb=4,
                    scale=3, channels=16, n_resblocks=1, weights=w_small, policy=pol, order=order)
    q.select(imp4)
    q.pack_step(imp4)
    print("policy", pol, "bins", q.host_results()["num_bins"])
from paper_2407_16990_b200.global_topk import global_select  # noqa: E402
global_select([(q, 0, imp4)], wl4.k, "cuda")
torch.cuda.synchronize()
t = rg.TemporalReuse(2, 30, 640, 360)
t.run(torch.from_numpy(synth.residuals_y(2, 30, 360, 640, 1)).cuda(), 12)
nv = torch.from_numpy(synth.frames_nv12(1, 2, 360, 640, 1)).cuda()
rgb = torch.empty((1, 2, 360, 640, 3), dtype=torch.uint8, device="cuda")
rg.nv12_to_rgb8(rg.Geom(1, 2, 640, 360, 16), nv, rgb)
torch.cuda.synchronize()
print("round-2 kernels ok")
