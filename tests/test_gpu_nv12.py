"""GPU parity of the NV12 input (regen_nv12_to_rgb8, reading D19): the conversion is
bit-exact against the oracle, and the hot path fed from NV12 produces exactly the HR frames of the
same path fed with the oracle-converted RGB8 frames."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("S,F,W,H", [(1, 30, 640, 360), (2, 3, 1280, 720), (1, 2, 320, 180), (1, 1, 4, 2)])
def test_nv12_conversion_bit_exact(S, F, W, H):
    import paper_2407_16990_b200 as rg
    nv = synth.frames_nv12(S, F, H, W, 3)
    out = torch.empty((S, F, H, W, 3), dtype=torch.uint8, device="cuda")
    rg.nv12_to_rgb8(rg.Geom(S, F, W, H, 16), torch.from_numpy(nv).cuda(), out)
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.nv12_to_rgb8(nv, W, H))


def test_pipeline_from_nv12_equals_pipeline_from_rgb():
    import paper_2407_16990_b200 as rg
    wl = synth.small(synth.CONFIGS["c2"], F=2)
    imp = torch.from_numpy(synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 4)).cuda()
    nv = synth.frames_nv12(wl.S, wl.F, wl.H, wl.W, 4)
    w = synth.sr_weights(wl.sr, 0)
    p = rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=128, bin_h=128, max_bins=wl.max_bins,
                    partition_mb=4, scale=3, channels=32, n_resblocks=8, weights=w)
    a = p.run(imp, p.convert_nv12(torch.from_numpy(nv).cuda())).clone()
    b = p.run(imp, torch.from_numpy(oracle.nv12_to_rgb8(nv, wl.W, wl.H)).cuda())
    assert torch.equal(a, b)


@pytest.mark.parametrize("W,H", [(640, 360), (200, 120)])
def test_nv12_frames_read_directly_equal_the_rgb_path(W, H):
    """geom.format = NV12: the gather and both bilinear kernels convert while reading (BT.601 fused, D19);
    every call's HR frames equal the RGB8 path on the oracle-converted frames, bit for bit (fused call,
    the two halves, and the separate enhance + scatter_blend with the row kernel)."""
    import dataclasses
    import paper_2407_16990_b200 as rg
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=2), W=W, H=H)
    imp = torch.from_numpy(synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 5)).cuda()
    nv = synth.frames_nv12(wl.S, wl.F, wl.H, wl.W, 5)
    rgb = torch.from_numpy(oracle.nv12_to_rgb8(nv, W, H)).cuda()
    nv = torch.from_numpy(nv).cuda()
    w = synth.sr_weights(wl.sr, 0)

    def pipe(fmt):
        return rg.Pipeline(S=wl.S, F=wl.F, W=W, H=H, k=wl.k, bin_w=128, bin_h=128, max_bins=wl.max_bins,
                           partition_mb=4, scale=3, channels=32, n_resblocks=wl.sr.n_resblocks, weights=w,
                           frame_format=fmt)
    pr, pn = pipe(rg.FORMAT_RGB8), pipe(rg.FORMAT_NV12)
    ref = pr.run(imp, rgb).clone()
    assert torch.equal(pn.run(imp, nv), ref)
    out = torch.full_like(ref, float("nan"))
    pn.scatter_bilinear(nv, out=out)
    pn.enhance_owned(nv, out=out)
    assert torch.equal(out, ref)
    assert torch.equal(pn.run(imp, nv, fused=False), pr.run(imp, rgb, fused=False))
