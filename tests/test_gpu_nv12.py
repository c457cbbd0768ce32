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
