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
