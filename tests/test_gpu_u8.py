"""u8 output frames (REGEN_DTYPE_U8, reading D20) through the C-ABI vs the oracle's quantised frames
(oracle.quantize_u8, pinned in test_oracle_u8.py):
- bilinear pixels are an exact integer function of the u8 frames: bit-exact;
- enhanced (pasted) pixels are the quantised model value: within 6 codes of the quantised fp64
  oracle (|dv| <= 2e-2 -> |d(255 v)| <= 5.1 -> rounded codes differ by <= 6), and EXACTLY
  clamp(rhe(255 * v)) of the same run's bf16 output v (the fused fold, the split calls and the
  separate enhance + blend calls all quantise the same bf16 value);
- every pixel is written exactly once (0- and 255-filled buffers give the same frames)."""
import dataclasses

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

U8_CODES = 6


def _rg():
    import paper_2407_16990_b200 as rg
    return rg


def _pipe(wl, w, **kw):
    rg = _rg()
    return rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=wl.bin_w, bin_h=wl.bin_h,
                       max_bins=wl.max_bins, partition_mb=wl.partition_mb, scale=wl.sr.scale,
                       channels=wl.sr.channels, n_resblocks=wl.sr.n_resblocks, weights=w, bf16=wl.sr.bf16,
                       res_scale=wl.sr.res_scale, **kw)


def _check(wl, seed, kind="blobs", nv12=False):
    rg = _rg()
    imp = synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, seed, kind)
    fr = synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, seed)
    w = synth.sr_weights(wl.sr, seed)
    kw = {}
    fr_in = fr
    if nv12:
        fr_in = synth.frames_nv12(wl.S, wl.F, wl.H, wl.W, seed)
        fr = oracle.nv12_to_rgb8(fr_in, wl.W, wl.H)
        kw = dict(frame_format=rg.FORMAT_NV12)
    imp_t, fr_t = torch.from_numpy(imp).cuda(), torch.from_numpy(fr_in).cuda()
    p8 = _pipe(wl, w, out_dtype=rg.DTYPE_U8, **kw)
    pn = _pipe(wl, w, **kw)                                   # the model dtype's frames, same inputs
    ref_native = pn.run(imp_t, fr_t).clone()
    p8.out.fill_(0)
    out = p8.run(imp_t, fr_t).clone()                          # regen_enhance_scatter
    p8.out.fill_(255)
    assert torch.equal(p8.run(imp_t, fr_t), out), "a pixel was not written (0- vs 255-filled buffers differ)"
    split = torch.full_like(out, 7)
    p8.scatter_bilinear(fr_t, out=split)
    p8.enhance_owned(fr_t, out=split)
    assert torch.equal(split, out), "regen_enhance_owned + regen_scatter_bilinear differ from the fused call"
    sep = p8.run(imp_t, fr_t, out=torch.full_like(out, 9), fused=False)   # enhance_packed + scatter_blend
    assert torch.equal(sep, out), "regen_enhance_packed + regen_scatter_blend differ from the fused call"
    g = p8.host_results()
    assert g["status"] == 0
    o = oracle.index_path(imp, wl.W, wl.H, wl.k, partition_mb=wl.partition_mb, bin_w=wl.bin_w, bin_h=wl.bin_h,
                          max_bins=wl.max_bins)
    np.testing.assert_array_equal(g["owner"], o["owner"])
    s = wl.sr.scale
    got = out.cpu().numpy().reshape(-1, s * wl.H, s * wl.W, 3)
    nat = ref_native.float().cpu().numpy().reshape(got.shape)
    owned_mb = (o["owner"] >= 0).reshape(-1, wl.GH, wl.GW)
    owned = np.repeat(np.repeat(owned_mb, 16 * s, 1), 16 * s, 2)[:, :s * wl.H, :s * wl.W]
    # enhanced pixels: exactly the quantised model-dtype value of the same run
    q_nat = np.round(np.clip(nat.astype(np.float64), 0.0, 1.0) * 255.0).astype(np.uint8)   # exact product
    np.testing.assert_array_equal(got[owned], q_nat[owned])
    lr = oracle.gather(fr, o["boxes"], o["placement"], wl.bin_w, wl.bin_h, o["num_bins"], wl.sr.bf16)
    hr = oracle.enhance(wl.sr, oracle.sr_weights_for(wl.sr, w), lr, o["boxes"], o["placement"],
                        threads=oracle.host_cores())
    ref64 = oracle.scatter(fr, o["boxes"], o["placement"], o["owner"], hr, s, wl.bin_w, wl.bin_h,
                           threads=oracle.host_cores())
    ref = oracle.quantize_u8(fr, o["owner"], ref64, s)
    np.testing.assert_array_equal(got[~owned], ref[~owned])
    d = np.abs(got.astype(np.int32) - ref.astype(np.int32))
    assert d.max() <= U8_CODES, f"enhanced pixels differ by {d.max()} codes"
    return int(owned.sum()), int((~owned).sum())


def test_u8_frames_c2_geometry():
    n_own, n_bil = _check(synth.small(synth.CONFIGS["c2"], F=2), 31)
    assert n_own > 0 and n_bil > 0


def test_u8_frames_x2_c5_network():
    """x2 (p = 2 fold, C = 64 unfused convs), 720p frames, 10% of the MBs."""
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c5"], F=1), S=1, pct=10.0, max_bins=128)   # ~10 bins used
    _check(wl, 32)


def test_u8_frames_fp32_model():
    """C1: the fp32 model (no fold): enhanced pixels come from the fp32 HR bins."""
    _check(synth.small(synth.CONFIGS["c1"], F=2), 33)


def test_u8_frames_nv12_input():
    """NV12 frames (the bilinear pass takes the row kernel with its integer u8 horizontal pass)."""
    _check(synth.small(synth.CONFIGS["c2"], F=2), 34, nv12=True)


@pytest.mark.parametrize("W,H", [(200, 120), (328, 184)])
def test_u8_frames_odd_sizes(W, H):
    """Widths that are not a multiple of 8 (row kernel, byte copy-out for unaligned rows) and partial MBs."""
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=2), W=W, H=H, pct=25.0,
                             sr=synth.SRConfig(3, 16, 1, 1.0, True))
    _check(wl, 35, kind="noisy")


@pytest.mark.parametrize("scale", [2, 4])
def test_u8_frames_even_scales_with_ties(scale):
    """x2 / x4: exact .5 ties occur in the bilinear pixels and must round to even like the oracle."""
    wl = dataclasses.replace(synth.small(synth.CONFIGS["c2"], F=1), sr=synth.SRConfig(scale, 16, 1, 1.0, True))
    _check(wl, 36 + scale)
