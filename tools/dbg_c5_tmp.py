import sys, os, dataclasses
sys.path.insert(0, os.getcwd())
import torch, numpy as np, synth
import paper_2407_16990_b200 as rg
for pct in (15.0, 25.0, 50.0):
    wl = dataclasses.replace(synth.CONFIGS["c5"], pct=pct, F=10)
    p = rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=128, bin_h=128, max_bins=wl.max_bins, partition_mb=4,
                    scale=2, channels=64, n_resblocks=16, weights=synth.sr_weights(wl.sr, 0))
    for g in range(4):
        imp = torch.from_numpy(synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 0, s0=2 * g)).cuda()
        fr = torch.from_numpy(synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, 0, s0=2 * g)).cuda()
        a = p.run(imp, fr).clone(); b = p.run(imp, fr).clone()
        print(pct, g, "nan", int(torch.isnan(a.float()).sum()), "equal", torch.equal(a, b), flush=True)
