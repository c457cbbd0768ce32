import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2407_16990_b200 as rg
wl = synth.CONFIGS["c1"]
imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 5)
fr = synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, 5)
w = synth.sr_weights(wl.sr, 5)
p = rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=wl.bin_w, bin_h=wl.bin_h, max_bins=wl.max_bins,
                partition_mb=wl.partition_mb, scale=wl.sr.scale, channels=wl.sr.channels, n_resblocks=wl.sr.n_resblocks,
                weights=w, bf16=wl.sr.bf16)
it, ft = torch.from_numpy(imp).cuda(), torch.from_numpy(fr).cuda()
out = p.run(it, ft, fused=False).clone()
o2 = torch.full_like(out, float("nan"))
p.scatter_bilinear(ft, out=o2)
p.enhance_owned(ft, out=o2)
d = (o2 != out)
print("diff count", int(d.sum()), "nan", int(torch.isnan(o2).sum()))
idx = torch.nonzero(d)[:10]
for r in idx.tolist():
    print(r, float(out[tuple(r)]), float(o2[tuple(r)]))
own = p.host_results()["owner"]
if len(idx):
    s_, f_, Y, X, c = idx[0].tolist()
    print("owner at", own[s_, f_, Y // 32, X // 32])
